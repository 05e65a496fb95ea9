#!/bin/bash
# Every bench workload, our arm then the reference arm (measurement tool):
#   bash tools/bench_all.sh <round tag>   -> gpurun_out/<tag>_bench_<workload>{,_reference}.json
tag=${1:-r02}
for wl in cfg4 cfg2 cfg3 cfg5 cfg5_u64 flag flagmix; do
  python bench.py --workload $wl > gpurun_out/${tag}_bench_${wl}.log 2>&1
  tail -1 gpurun_out/${tag}_bench_${wl}.log > gpurun_out/${tag}_bench_${wl}.json
  python bench.py --workload $wl --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_${wl}_reference.log 2>&1
  tail -1 gpurun_out/${tag}_bench_${wl}_reference.log > gpurun_out/${tag}_bench_${wl}_reference.json
done
