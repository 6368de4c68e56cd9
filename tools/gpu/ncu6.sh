mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_log_diff|k_exact" -s 0 -c 3 -o gpurun_out/prof_log -f python tools/gpu/prof_kernels.py 1024 log 2>&1 | tail -1
ncu -i gpurun_out/prof_log.ncu-rep --page source --csv > gpurun_out/log_src.csv 2>/dev/null
