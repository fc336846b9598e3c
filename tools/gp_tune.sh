mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_tuner.py -m gpu -q -x -k "filter or tune or explicit" > gpurun_out/pytest_q.log 2>&1; echo rc=$? >> gpurun_out/pytest_q.log
timeout 900 python tools/tune_time.py > gpurun_out/tune_time.jsonl 2> gpurun_out/tune_time.err
