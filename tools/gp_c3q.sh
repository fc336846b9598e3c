# config 3 check: a 2-minute smoke of the convolution pass first (hang guard), staged-engine
# parity tests + full-size config 3, bench (no tune) x2
set -u
mkdir -p gpurun_out
timeout 120 python tools/run_config.py --config 3 --steps 2 > gpurun_out/c3_plain.log 2>&1; rc=$?; echo "plain rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "s512 or merged or staged or conv9 or real_path or config3 or graph or window" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
timeout 400 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "config3" >> gpurun_out/pytest_q.log 2>&1; echo "pytest_full rc=$?" >> gpurun_out/pytest_q.log
for i in 1 2; do
  timeout 200 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/c3_$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/c3_$i.json').read().strip().splitlines()[-1]); print('run $i', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['whole_step']['per_kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done
