# A/B on one box: W8 convolution pass with / without the folder warps (config 3, fixed plan)
set -u
mkdir -p gpurun_out
timeout 120 python tools/run_config.py --config 3 --steps 2 > gpurun_out/c3_plain.log 2>&1; rc=$?; echo "plain rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
for i in 1 2 3; do
  for v in 0 1; do
    if [ $v = 1 ]; then export HD_S512_NOFOLDW=1; else unset HD_S512_NOFOLDW; fi
    timeout 200 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/fw_$v.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/fw_$v.json').read().strip().splitlines()[-1]); print('nofoldw=$v', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['whole_step']['per_kernel_ms'].items()}, d['clocks']['sm_mhz'])"
  done
done
