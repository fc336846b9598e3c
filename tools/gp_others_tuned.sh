# configs 2, 4, 5 with the tuner's plans (bench default tuning) -> gpurun_out/other_tuned_r02.jsonl
set -u
mkdir -p gpurun_out
rm -f gpurun_out/other_tuned_r02.jsonl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for C in 2 4 5; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-e2e --no-explicit 2>> gpurun_out/other_tuned_r02.err | tail -1 >> gpurun_out/other_tuned_r02.jsonl
done
