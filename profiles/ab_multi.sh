# bench the same workload from several build dirs on one box: bash profiles/ab_multi.sh config steps dir...
B='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])'
cfg=$1; st=$2; shift 2
for dir in "$@"; do echo -n "$dir $cfg: "; (cd $dir && python bench.py --steps $st --warmup 5 --config $cfg --no-cpu-baseline --no-e2e 2>/dev/null | python -c "$B"); done
