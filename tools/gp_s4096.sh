# 1-D m = 4096 engine check: its parity tests, config 2 with the new default (s4096r)
# against the m = 2048 engine (HD_NO_S4096R=1), then ncu of the new pass
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "s4096r or s2048r or s512c" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
python bench.py --config 2 --steps 20 --warmup 3 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
HD_NO_S4096R=1 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/bench_c2_old.json 2>> gpurun_out/bench_c2.err
if [ "${HD_NCU:-1}" = 1 ]; then
ncu --set full --clock-control none --import-source on -k regex:"s4096r" -s 1 -c 1 -o gpurun_out/prof_c2_4096 python tools/run_config.py --config 2 --steps 2 > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
fi
