#!/bin/bash
# bench (default) + its launch list + ncu --set full of the headline kernels; $1 = tag
tag=${1:-x}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$tag.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --workload headline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gauss_tri|k_median3_f32|k_box_stream' -c 3 -o gpurun_out/full_$tag -f python tools/gpu/prof_headline.py 1024 gmM > gpurun_out/full_$tag.log 2>&1
tail -1 gpurun_out/bench_$tag.log; grep '^{' gpurun_out/bench_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline'], d['filters'])"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_morph_bits2 -c 1 -o gpurun_out/full_${tag}_mbits -f python tools/gpu/prof_morph_bits.py > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_morph_u16s -c 1 -o gpurun_out/full_${tag}_mu16 -f python tools/gpu/prof_morph_u16.py > /dev/null 2>&1
