ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/slab_launches.csv python tools/slab_host.py > gpurun_out/slab_ncu.log 2>&1
echo rc=$?
