# TMA for jd-tiled inputs (slab exchanges at N > 1): dist tests (emulated ranks), staged parity, per-rank stage times
set -u
mkdir -p gpurun_out
rm -f gpurun_out/pytest_q.log
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_layouts.py -m gpu -x -q -k "${HD_TESTS:-dist or slab or s512 or merged or staged or conv9 or window or layouts or pass}" >> gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
HD_DEBUG_LAUNCH=1 timeout 600 python tools/slab_stage_times.py > gpurun_out/slab_stages.txt 2> gpurun_out/slab_stages.err; echo "stages rc=$?" >> gpurun_out/pytest_q.log
