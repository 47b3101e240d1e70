#!/bin/bash
# Generic bench A/B: ab_env.sh TAG "configs" "arm1" "arm2" ... where each arm is a space-separated
# list of VAR=value env settings ("-" = defaults).  Two alternating rounds per config.
T=$1; CONFIGS=$2; shift 2
for c in $CONFIGS; do
  for rep in 1 2; do
    for arm in "$@"; do
      envs=""; [ "$arm" != "-" ] && envs="$arm"
      line=$(env $envs timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1)
      echo "$line" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '[$arm]', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/${T}_bench.txt 2>&1 || echo "$c [$arm] FAILED" >> gpurun_out/${T}_bench.txt
    done
  done
done
