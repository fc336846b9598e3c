# ncu --set full of config 4's z convolution pass and config 5's multi-pair pass (default plans)
set -u
mkdir -p gpurun_out
ncu --set full --clock-control none -k regex:"^s128_kernel" -s 3 -c 1 -o gpurun_out/prof_c4z python tools/run_config.py --config 4 --steps 2 > gpurun_out/ncu_c4z.log 2>&1; echo "c4 rc=$?"
ncu --set full --clock-control none -k regex:"mconv" -s 0 -c 1 -o gpurun_out/prof_c5 python tools/run_config.py --config 5 --steps 2 > gpurun_out/ncu_c5.log 2>&1; echo "c5 rc=$?"
