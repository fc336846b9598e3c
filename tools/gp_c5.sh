# config 5 check: multi-pair parity tests, default-plan line (x3)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "multi or mconv or pair" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
for i in 1 2 3; do
  python bench.py --config 5 --steps 20 --warmup 3 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/c5_$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/c5_$i.json').read().strip().splitlines()[-1]); print('run $i', round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['whole_step']['per_kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done
