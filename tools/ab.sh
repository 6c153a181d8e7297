#!/bin/bash
# dev helper: A/B bench of two builds of libltfb_gpu.so (tools/ab/lib_base.so vs lib_new.so),
# interleaved runs, prints ms_per_step of each. Usage (on the GPU box): tools/ab.sh [reps] [extra bench args]
R=${1:-3}; shift
for i in $(seq 1 $R); do
  for v in base new; do
    LTFB_LIB_PATH=$PWD/tools/ab/lib_$v.so python bench.py --steps 2000 --warmup 5 --no-cpu-baseline "$@" 2>/dev/null \
      | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', round(d['ms_per_step']*1000,2), {k: round(v*1000,1) for k,v in d['kernels_ms_per_launch'].items() if v})"
  done
done
