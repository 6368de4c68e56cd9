#!/bin/bash
# end-of-round evidence in one call: bench line + launch list + ncu --set full
# of the headline / morphology kernels, summarised on the box (ncu reports
# themselves are too large to bring back); $1 = tag
tag=${1:-x}
bash tools/gpu/r02_bench_prof.sh $tag
for r in full_$tag full_${tag}_mbits full_${tag}_mu16; do
  [ -f gpurun_out/$r.ncu-rep ] || continue
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep gpurun_out/sum_$r.md > /dev/null 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$r.csv 2>/dev/null
  gzip -f gpurun_out/src_$r.csv
done
cp profiles/traffic.json gpurun_out/traffic_$tag.json
rm -f gpurun_out/*.ncu-rep
