#!/bin/bash
# Adaptive segmented kernel: tile-mode depth / load width (measurement tool; tuning build).
# (The SGAT variants it names were removed after the measurement, profiles/r02_seg_tile_depth_vb.txt.)
#   bash tools/seg_tile_vb.sh > gpurun_out/seg_tile_vb.txt
export POSPOP_LIBRARY=tuning
run() {
  local label=$1 wl=$2; shift 2
  env "$@" python bench.py --workload $wl --steps 100 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$label', '$wl', d['value'], d['ms_per_step'], r.get('kernel_ms_single_launch'))"
}
for rep in 1 2; do
  run default cfg5 POSPOP_X=1
  for v in "5,32,8" "6,32,8" "6,16,8"; do run "$v" cfg5 POSPOP_SEG_VARIANT=$v; done
  run default cfg5_u64 POSPOP_X=1
  for v in "5,32,8" "6,16,8"; do run "$v" cfg5_u64 POSPOP_SEG_VARIANT=$v; done
done
