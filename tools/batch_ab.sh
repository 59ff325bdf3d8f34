#!/bin/bash
# A/B of batch-kernel builds: FABM_LIBRARY=build_ab/libfabm_<v>.so, T=512 (the 8-GPU share) and T=4096
for v in "$@"; do
  for T in 512 4096; do
    echo -n "== $v T=$T: "
    FABM_LIBRARY=build_ab/libfabm_$v.so timeout 300 python bench.py --workload batch --batch-size $T --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=[json.loads(l) for l in sys.stdin if l.startswith('{')][0]; print(round(d['ms_per_step'],1), 'ms frac', round(d['roofline']['frac'],4), 'checksum', d['y_N_checksum'])"
  done
done
