# cfg5 sweep of the warp-per-array tile kernels (sched 11 strided, 12 CTA-blocked,
# 13 strided + first array read before the PDL wait) against the default
# adaptive kernel (empty variant).  Run on the GPU box.
for v in "7,32,13,1" "6,32,13,1" "6,32,13,2" "7,32,11,1" ""; do
  POSPOP_LIBRARY=tuning POSPOP_SEG_VARIANT=$v python bench.py --workload cfg5 --steps 50 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('u32', '$v', d['value'], d['roofline']['kernel_ms_isolated'])"
done
for v in "6,32,13,1" "6,32,11,1" ""; do
  POSPOP_LIBRARY=tuning POSPOP_SEG_VARIANT=$v python bench.py --workload cfg5_u64 --steps 50 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('u64', '$v', d['value'], d['roofline']['kernel_ms_isolated'])"
done
