# ncu --set full of config 3's convolution pass (default plan) -> gpurun_out/prof_conv.ncu-rep
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PLAN='[{"m":512,"C":1,"S":4,"D":9,"threads":0},{"m":512,"C":1,"S":8,"D":9,"threads":0}]'
python tools/run_config.py --config 3 --steps 2 --plan "$PLAN" > gpurun_out/plain_conv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"s512" -s 4 -c 1 -o gpurun_out/prof_conv python tools/run_config.py --config 3 --steps 2 --plan "$PLAN" > gpurun_out/ncu_conv.log 2>&1
echo ncu rc=$?
