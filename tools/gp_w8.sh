# W8 (8 compute warps at 232 registers) check: per-pass A/B, staged parity (both masks), full-size config 3, bench
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PLAN='[[{"m":512,"C":1,"S":16,"D":9,"threads":0},{"m":512,"C":1,"S":2,"D":9,"threads":0}]]'
for W in 2 0 3; do
  HD_S512_W8=$W timeout 300 python tools/pass_times.py --config 3 --plans "$PLAN" >> gpurun_out/pass_times.log 2>&1
done
K="${HD_TESTS:-s512 or merged or multipair or real_path or staged or slab or conv9 or filter or window}"
for W in ${HD_W8_TEST:-2 3}; do
  HD_S512_W8=$W timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q -k "$K" >> gpurun_out/pytest_q.log 2>&1; echo "pytest W8=$W rc=$?" >> gpurun_out/pytest_q.log
  HD_S512_W8=$W timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "config3" >> gpurun_out/pytest_q.log 2>&1; echo "pytest_full W8=$W rc=$?" >> gpurun_out/pytest_q.log
done
