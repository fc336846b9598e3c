# config 2 timing repeats (default plan), optional env in $1
set -u
mkdir -p gpurun_out
for i in 1 2 3; do
  python bench.py --config 2 --steps 20 --warmup 3 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/ab_$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ab_$i.json').read().strip().splitlines()[-1]); print('run $i', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
