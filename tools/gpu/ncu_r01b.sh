# full-set capture of every hot kernel (one launch each) + the bench launch list
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_median3|k_box_stream|k_gauss_p2|k_exact|k_log_stream|k_morph3" -c 9 -o gpurun_out/prof_r01b -f python tools/gpu/prof_all.py 1024 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_under_ncu.txt 2>&1
