mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gauss_x2" -s 1 -c 1 -o gpurun_out/prof_gx2 -f python tools/gpu/prof_kernels.py 1024 gauss 2>&1 | tail -1
ncu -i gpurun_out/prof_gx2.ncu-rep --page source --csv > gpurun_out/gx2_src.csv 2>/dev/null
