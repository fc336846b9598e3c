# slab path check: dist tests (world 1 + emulated ranks) and the config-3 slab bench line at world 1
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.log
timeout 600 python bench.py --config 3 --mode slab --steps 50 --warmup 5 --no-cpu --no-explicit --no-tune > gpurun_out/bench_slab.json 2> gpurun_out/bench_slab.err; echo "bench rc=$?"
HD_DEBUG_LAUNCH=1 timeout 300 python bench.py --config 3 --mode slab --steps 3 --warmup 3 --no-cpu --no-explicit --no-tune --no-e2e > /dev/null 2> gpurun_out/slab_launch.err
