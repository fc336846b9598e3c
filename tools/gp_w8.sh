# W8 (8 compute warps at 232 registers) check: staged parity, full-size config 3, per-pass A/B, bench
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PLAN='[[{"m":512,"C":1,"S":16,"D":9,"threads":0},{"m":512,"C":1,"S":2,"D":9,"threads":0}]]'
timeout 300 python tools/pass_times.py --config 3 --plans "$PLAN" > gpurun_out/pass_times.log 2>&1; echo "pt rc=$?" >> gpurun_out/pass_times.log
HD_S512_W8=0 timeout 300 python tools/pass_times.py --config 3 --plans "$PLAN" >> gpurun_out/pass_times.log 2>&1
HD_S512_W8=7 timeout 300 python tools/pass_times.py --config 3 --plans "$PLAN" >> gpurun_out/pass_times.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q -k "${HD_TESTS:-s512 or merged or multipair or real_path or staged or slab or conv9 or filter or window}" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "config3" >> gpurun_out/pytest_q.log 2>&1; echo "pytest_full rc=$?" >> gpurun_out/pytest_q.log
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
