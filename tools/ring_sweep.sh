#!/bin/bash
# Sweep the persistent 2D kernel's ring geometry (GRFC_RING_LA / GRFC_RING_SL) on one config.
cd "$(dirname "$0")/.."
for cfg in ${SWEEP:-12_8 6_4 4_3 4_4 3_3 5_3}; do
  cfg=${cfg//_/ }
  set -- $cfg
  r=$(GRFC_RING_LA=$1 GRFC_RING_SL=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f Gpts/s' % d['value'])" 2>&1 | tail -1)
  echo "LA=$1 SL=$2: $r"
done
