# per-phase cycles of the staged m = 512 passes (config 3): a separate build with
# -DHD_PHASE_PROF_BUILD (objects rebuilt from scratch), HD_PHASE_PROF=1 at run time
mkdir -p gpurun_out
rm -rf paper_2306_10016_b200/csrc/build
NVCC_APPEND_FLAGS=-DHD_PHASE_PROF_BUILD python -m paper_2306_10016_b200.build --force > gpurun_out/build_phase.log 2>&1
PLAN='[{"m":512,"C":1,"S":16,"D":9,"threads":0},{"m":512,"C":1,"S":2,"D":9,"threads":0}]'
HD_PHASE_PROF=1 python tools/run_config.py --config 3 --steps 2 --plan "$PLAN" > gpurun_out/phase.log 2>&1
HD_S512_W8=3 HD_PHASE_PROF=1 python tools/run_config.py --config 3 --steps 2 --plan "$PLAN" >> gpurun_out/phase.log 2>&1
