# ncu --set full (with source) of one config-3 step (fwd_x, conv_y, inv_x) with the bench's tuned plan
set -u
mkdir -p gpurun_out
PLAN='[{"m":512,"C":1,"S":8,"D":9,"threads":0},{"m":512,"C":1,"S":16,"D":9,"threads":0}]'
python tools/run_config.py --config 3 --steps 2 --plan "$PLAN" > gpurun_out/plain_step.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"s512" -s 3 -c 3 -o gpurun_out/prof_step python tools/run_config.py --config 3 --steps 2 --plan "$PLAN" > gpurun_out/ncu_step.log 2>&1
echo ncu rc=$?
