# usage: bash tools/gpu/test_bench.sh [pytest-args]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -q -m gpu -x "$@" 2>&1 | tail -25 > gpurun_out/pytest_gpu.txt; tail -25 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 --extra --no-cpu 2>&1 | tail -3 | tee gpurun_out/bench.txt
