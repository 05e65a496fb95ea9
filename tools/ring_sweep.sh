#!/bin/bash
# Ring kernel (SCHED 6) vs the LDG kernel (measurement tool; tuning build).
#   bash tools/ring_sweep.sh > gpurun_out/ring_sweep.txt
export POSPOP_LIBRARY=tuning
run() {  # label, workload, env...
  local label=$1 wl=$2; shift 2
  env "$@" python bench.py --workload $wl --steps 50 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$label', '$wl', d['value'], d['ms_per_step'], r.get('kernel_ms_single_launch'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
for wl in flag flagmix; do
  run ldg $wl POSPOP_X=1
  for rv in "5,32,0,512,6,2 16,1" "5,32,0,512,6,2 24,1,1" "5,32,0,512,6,2 20,1,1" "5,32,0,512,6,2 16,1,1" "5,32,0,512,6,2 12,2,1" "4,32,0,512,6,2 24,2,1" "4,32,0,512,6,2 32,1,1"; do
    set -- $rv
    run "ring $1 $2" $wl POSPOP_FLAG_VARIANT=$1 POSPOP_RING=$2
  done
done
for wl in ${RING_COUNT_WL:-}; do
  run ldg $wl POSPOP_X=1
  for rv in "7,32,0,256,6 8,1" "7,32,0,256,6 4,3" "6,32,0,256,6 16,1" "6,32,0,256,6 12,2"; do
    set -- $rv
    run "ring $1 $2" $wl POSPOP_STREAM_VARIANT=$1 POSPOP_RING=$2
  done
done
