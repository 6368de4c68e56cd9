# round-1 evidence: default bench line, --extra breakdown, ncu full-set (two
# captures, <64 MiB each) and the launch list of the default bench command
mkdir -p gpurun_out
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_final.json
timeout 600 python bench.py --steps 5 --warmup 3 --extra --no-cpu 2>&1 | tail -1 > gpurun_out/bench_extra_final.json
timeout 600 ncu --set full --clock-control none -k regex:"k_median3|k_box_stream|k_gauss_p2|k_morph3" -c 4 -o gpurun_out/prof_final1 -f python tools/gpu/prof_all.py 1024 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_exact|k_log_stream" -c 4 -o gpurun_out/prof_final2 -f python tools/gpu/prof_all.py 1024 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
ls -la gpurun_out
