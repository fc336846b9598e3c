# config 4 check: s128 parity tests, default-plan line (x2)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layouts.py -m gpu -x -q -k "s128 or c64 or 3d" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
for i in 1 2; do
  python bench.py --config 4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/c4_$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/c4_$i.json').read().strip().splitlines()[-1]); print('run $i', round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['whole_step']['per_kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done
