mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_median3|k_sep3d|k_morph3|k_exact|k_log_diff" -s 0 -c 7 -o gpurun_out/prof_r01_final -f python tools/gpu/prof_kernels.py 1024 median,mean,gauss,erode,log 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_final.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_under_ncu.txt 2>&1
