# A/B on one box: x passes nine-warp (default) vs W8 (HD_S512_W8=3), config 3 fixed plan
set -u
mkdir -p gpurun_out
for i in 1 2; do
  for v in 2 3; do
    HD_S512_W8=$v timeout 200 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/w8_$v.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/w8_$v.json').read().strip().splitlines()[-1]); print('W8=$v', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['whole_step']['per_kernel_ms'].items()}, d['clocks']['sm_mhz'])"
  done
done
