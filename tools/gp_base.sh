set -u
mkdir -p gpurun_out
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak) > gpurun_out/fp64_peak.json 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/fp64_peak.json
python bench.py --steps 200 --warmup 5 > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err
echo bench rc=$?
PLAN=$(python -c "import json;d=json.loads(open('gpurun_out/bench_base.json').read().strip().splitlines()[-1]);print(json.dumps([{k:a[k] for k in ('m','C','S','D','threads')} for a in d['config']['plan']]))")
ncu --set full --clock-control none --import-source on -k regex:"s512" -s 3 -c 3 -o gpurun_out/prof_base python tools/run_config.py --config 3 --steps 2 --plan "$PLAN" > gpurun_out/ncu_base.log 2>&1
echo ncu rc=$?
