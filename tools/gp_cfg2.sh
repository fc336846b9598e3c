# 1-D engine check: parity tests, config-2 bench line (default plan), ncu of its pass
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q -k "s2048r or s512c or batched_1d or lambda or dist or conv1d" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "config2" >> gpurun_out/pytest_q.log 2>&1; echo "pytest_full rc=$?" >> gpurun_out/pytest_q.log
python bench.py --config 2 --steps 20 --warmup 3 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"s2048r|pass_kernel" -s 1 -c 1 -o gpurun_out/prof_c2new python tools/run_config.py --config 2 --steps 2 > gpurun_out/ncu_c2new.log 2>&1; echo "ncu rc=$?"
