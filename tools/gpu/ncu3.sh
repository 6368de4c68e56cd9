mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_morph2" -s 1 -c 1 -o gpurun_out/prof_morph -f python tools/gpu/prof_kernels.py 1024 erode 2>&1 | tail -1
