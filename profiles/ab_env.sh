# bench one build under several environment settings: bash profiles/ab_env.sh config steps "ENV=.." ...
B='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])'
cfg=$1; st=$2; shift 2
for e in "$@"; do echo -n "[$e] $cfg: "; env $e python bench.py --steps $st --warmup 5 --config $cfg --no-cpu-baseline --no-e2e 2>/dev/null | python -c "$B"; done
