#!/bin/bash
# Runs ON the GPU box: the bench's graded apply (cfg2, 50 steps) for library
# variants, interleaved three times.   bash scripts/ab_apply.sh base ns6 ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
lib_of() { if [ "$1" = base ]; then echo $PWD/paper_2201_12931_b200/libvoxb200.so; else echo $PWD/paper_2201_12931_b200/libvoxb200_$1.so; fi; }
for rep in 1 2 3; do
  for t in "$@"; do
    VT_LIB_PATH=$(lib_of $t) timeout 300 python bench.py --no-cpu --simp-iters 0 --no-cfg5 --steps 50 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t apply', round(d['ms_per_step']*1e3,1),'us', round(d['value'],1),'GDOF/s frac', round(d['roofline']['frac'],3))"
  done
done
