mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sep3d|k_median|k_morph" -s 4 -c 4 -o gpurun_out/prof_r01_a -f python tools/gpu/prof_kernels.py 1024 2>&1 | tail -5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_a.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | tail -2
