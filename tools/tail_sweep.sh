#!/bin/bash
# Stream-kernel tail sweep (measurement tool; the tuning build's knobs):
# pool chunk size CB and pool tiles per warp vs single-launch and
# back-to-back time for cfg2 (512 MiB) and cfg4 (8 GiB).
#   bash tools/tail_sweep.sh > gpurun_out/tail_sweep.txt
export POSPOP_LIBRARY=tuning
for wl in cfg2 cfg4; do
  for cb in 2 1; do
    for ppw in 0 2 4 8; do
      POSPOP_CHUNK_B=$cb POSPOP_POOL_TILES_PER_WARP=$ppw python bench.py --workload $wl --steps 100 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$wl', 'cb=$cb', 'ppw=$ppw', d['value'], d['ms_per_step'], r.get('kernel_ms_single_launch'))"
    done
  done
done
