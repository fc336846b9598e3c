# the other BASELINE configs (default plans) and the slab path at world 1 -> gpurun_out/other_r02.jsonl
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for C in 2 4 5; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-e2e --no-explicit --no-tune 2>> gpurun_out/other_r02.err | tail -1 >> gpurun_out/other_r02.jsonl
done
timeout 600 python bench.py --config 3 --mode slab --steps 50 --warmup 5 --no-cpu --no-explicit --no-tune 2>> gpurun_out/other_r02.err | tail -1 >> gpurun_out/other_r02.jsonl
