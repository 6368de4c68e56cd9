mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_median3" -s 1 -c 1 -o gpurun_out/prof_med2 -f python tools/gpu/prof_kernels.py 1024 median 2>&1 | tail -1
ncu -i gpurun_out/prof_med2.ncu-rep --page source --csv > gpurun_out/med2_src.csv 2>/dev/null
ncu -i gpurun_out/prof_med2.ncu-rep --page details --csv > gpurun_out/med2_details.csv 2>/dev/null
