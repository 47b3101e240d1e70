# A/B of two builds on the same box: bash profiles/ab.sh DIR_A DIR_B [config] [steps]
B='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])'
cfg=${3:-metr_la}; st=${4:-300}
for i in 1 2; do for dir in "$1" "$2"; do echo -n "$dir $cfg: "; (cd $dir && python bench.py --steps $st --warmup 5 --config $cfg --no-cpu-baseline --no-e2e 2>/dev/null | python -c "$B"); done; done
