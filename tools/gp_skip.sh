mkdir -p gpurun_out; rm -f gpurun_out/pass_times.log
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PLAN='[[{"m":512,"C":1,"S":16,"D":9,"threads":0},{"m":512,"C":1,"S":16,"D":9,"threads":0}]]'
for S in 0 1 2 3; do echo "skip=$S" >> gpurun_out/pass_times.log; HD_DEBUG_SKIP=$S timeout 300 python tools/pass_times.py --config 3 --plans "$PLAN" >> gpurun_out/pass_times.log 2>&1; done
