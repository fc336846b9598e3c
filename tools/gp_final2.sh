# round-2 final evidence: full GPU suite, smoke, default bench line, its launch list and
# one ncu --set full step capture (tools/profile_bench.sh), other configs
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-explicit > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 bash tools/profile_bench.sh 3 r02f > gpurun_out/profile_bench.log 2>&1
