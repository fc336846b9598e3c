# full GPU suite + smoke + default bench + the other configs' default-plan lines
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
rm -f gpurun_out/other_r02.jsonl
for C in 2 4 5; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-e2e --no-explicit --no-tune 2>> gpurun_out/other_r02.err | tail -1 >> gpurun_out/other_r02.jsonl
done
