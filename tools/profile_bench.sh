#!/bin/bash
# One gpurun call: bench (default, tuned plan) -> plain run of that plan ->
# ncu launch list -> ncu --set full of one step's kernels.  Outputs in gpurun_out/.
# usage: tools/profile_bench.sh <config> <tag>
set -u
CFG=${1:-3}
TAG=${2:-r01}
mkdir -p gpurun_out
python bench.py --config "$CFG" --steps 200 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
PLAN=$(python -c "import json;d=json.loads(open('gpurun_out/bench_${TAG}.json').read().strip().splitlines()[-1]);print(json.dumps([{k:a[k] for k in ('m','C','S','D','threads')} for a in d['config']['plan']]))")
echo "plan $PLAN"
NK=$(python -c "print({1:1,2:1,3:3,4:7,5:4}[$CFG])")
python tools/run_config.py --config "$CFG" --steps 2 --plan "$PLAN" > gpurun_out/plain_${TAG}.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python tools/run_config.py --config "$CFG" --steps 2 --plan "$PLAN" > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"pass_kernel|s512" -s "$NK" -c "$NK" \
    -o gpurun_out/prof_${TAG} python tools/run_config.py --config "$CFG" --steps 2 --plan "$PLAN" > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"
