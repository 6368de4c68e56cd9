#!/bin/bash
# round-2 checkpoint: GPU tests, default bench, launch list of the bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --workload headline > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log
