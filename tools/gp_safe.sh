set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 180 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv9v3" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
grep -q "rc=0" gpurun_out/pytest_q.log && timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "s512_engine or merged or multipair or real_path or staged" >> gpurun_out/pytest_q.log 2>&1; echo "pytest2 rc=$?" >> gpurun_out/pytest_q.log
grep -q "pytest2 rc=0" gpurun_out/pytest_q.log && timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --no-explicit --no-tune > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
grep -q "pytest2 rc=0" gpurun_out/pytest_q.log && timeout 300 bash tools/gp_ncu_conv.sh
