# ncu --set full (with source) of config 4's z convolution pass (default plan)
set -u
mkdir -p gpurun_out
python tools/run_config.py --config 4 --steps 2 > gpurun_out/plain_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^s128_kernel" -c 6 -o gpurun_out/prof_c4conv python tools/run_config.py --config 4 --steps 2 > gpurun_out/ncu_c4.log 2>&1
echo ncu rc=$?
