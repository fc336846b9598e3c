# quick GPU check: p512 parity tests, config-3 full-size parity, a short bench, per-pass times
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "p512 or merged or s512_engine or graph or scratch or config3" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "config3_full" > gpurun_out/pytest_full3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full3.log
python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
HD_NO_P512=1 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --no-explicit > gpurun_out/bench_q_nop512.json 2>> gpurun_out/bench_q.err
