# A/B of a kernel change: per-pass times of config 3 (three runs) + staged parity + full-size config 3
set -u
mkdir -p gpurun_out
rm -f gpurun_out/pass_times.log gpurun_out/pytest_q.log
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PLAN='[[{"m":512,"C":1,"S":16,"D":9,"threads":0},{"m":512,"C":1,"S":16,"D":9,"threads":0}]]'
for i in 1 2 3; do timeout 300 python tools/pass_times.py --config 3 --plans "$PLAN" >> gpurun_out/pass_times.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layouts.py -m gpu -x -q -k "${HD_TESTS:-s512 or merged or multipair or real_path or staged or conv9 or window or layouts or residue or fft}" >> gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "config3" >> gpurun_out/pytest_q.log 2>&1; echo "pytest_full rc=$?" >> gpurun_out/pytest_q.log
