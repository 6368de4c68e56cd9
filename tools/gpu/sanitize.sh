mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/gpu/sanitize.py > gpurun_out/san_memcheck.txt 2>&1; tail -3 gpurun_out/san_memcheck.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/gpu/sanitize.py > gpurun_out/san_racecheck.txt 2>&1; tail -3 gpurun_out/san_racecheck.txt
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python tools/gpu/sanitize.py > gpurun_out/san_synccheck.txt 2>&1; tail -3 gpurun_out/san_synccheck.txt
