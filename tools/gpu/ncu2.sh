mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sep3d|k_median" -s 3 -c 3 -o gpurun_out/prof_r01_b -f python tools/gpu/prof_kernels.py 1024 median,mean,gauss 2>&1 | tail -2
