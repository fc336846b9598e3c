# ncu --set full of one step of configs 2 and 5 (default plans) + launch lists
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for C in 2 5; do
  python tools/run_config.py --config $C --steps 2 > gpurun_out/plain_c$C.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$C.csv python tools/run_config.py --config $C --steps 2 > /dev/null 2>&1
  NK=$([ $C = 2 ] && echo 1 || echo 4)
  ncu --set full --clock-control none --import-source on -k regex:"pass_kernel|s512" -s $NK -c $NK -o gpurun_out/prof_c$C python tools/run_config.py --config $C --steps 2 > gpurun_out/ncu_c$C.log 2>&1
  echo "config $C ncu rc=$?"
done
