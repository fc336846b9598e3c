# iteration check: staged-engine parity tests, per-pass bench times, ncu of the conv pass
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${HD_TESTS:-s512_engine or merged or multipair or real_path or staged or conv9}" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
bash tools/gp_ncu_conv.sh
