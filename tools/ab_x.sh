#!/bin/bash
# A/B the free-form variant libraries (build/libgrfc_x*.so) on config c2.
cd "$(dirname "$0")/.."
for lib in paper_1105_2737_b200/lib/libgrfc.so paper_1105_2737_b200/build/libgrfc_x*.so; do
  r=$(GRFC_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} 2>&1 | tail -1 |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f Gpts/s' % d['value'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" 2>&1 | tail -1)
  echo "$lib: $r"
done
