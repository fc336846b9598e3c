# GPU check of the distributed entry points (world 1 + emulated ranks) and a slab-mode bench
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
#timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.log
python bench.py --mode slab --steps 20 --warmup 3 --no-cpu --no-explicit --no-tune > gpurun_out/bench_slab.json 2> gpurun_out/bench_slab.err; echo "slab rc=$?"
python bench.py --mode slab --config 4 --steps 10 --warmup 3 --no-cpu --no-explicit --no-tune > gpurun_out/bench_slab4.json 2>> gpurun_out/bench_slab.err; echo "slab4 rc=$?"
