#!/bin/bash
# ncu --set full of the two headline kernels (gaussian ws sigma=2, median r=1) on the bench's 1024^3 block
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gauss_tri|k_gauss_ws|k_median3_f32|k_median3_plane' -c 2 \
  -o gpurun_out/headline_${1:-a} -f python tools/gpu/prof_headline.py 1024 ${2:-gm} > gpurun_out/prof_${1:-a}.log 2>&1
tail -3 gpurun_out/prof_${1:-a}.log
