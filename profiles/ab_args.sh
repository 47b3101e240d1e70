# bench extra args from several build dirs on one box: bash profiles/ab_args.sh "ARGS" steps dir...
B='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])'
args=$1; st=$2; shift 2
for dir in "$@"; do echo -n "$dir [$args]: "; (cd $dir && python bench.py --steps $st --warmup 5 $args --no-cpu-baseline --no-e2e 2>/dev/null | python -c "$B"); done
