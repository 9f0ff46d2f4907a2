#!/bin/bash
# Dev helper (runs ON the GPU box): A/B the apply kernel of the built library variants.
#   bash scripts/ab.sh tag1 tag2 ...   ("" = the default libvoxb200.so)
for t in "$@"; do
  if [ "$t" = "base" ]; then lib=paper_2201_12931_b200/libvoxb200.so; else lib=paper_2201_12931_b200/libvoxb200_$t.so; fi
  for rep in 1 2; do
    VT_LIB_PATH=$PWD/$lib python bench.py --no-cpu --simp-iters 0 --steps 50 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['ms_per_step']*1e3,1),'us', round(d['value'],1),'GDOF/s frac', round(d['roofline']['frac'],3))"
  done
done
