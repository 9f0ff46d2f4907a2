#!/bin/bash
# Runs ON the GPU box: A/B the hex8 variants (tags of _build.py; "base" = the
# default libvoxb200.so): apply timing via the bench, kernel timings via
# quick_apply, and the operator / solver parity tests against each variant.
#   bash scripts/ab_hex8.sh base z2 z2t12 ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for t in "$@"; do
  if [ "$t" = "base" ]; then lib=$PWD/paper_2201_12931_b200/libvoxb200.so; else lib=$PWD/paper_2201_12931_b200/libvoxb200_$t.so; fi
  for rep in 1 2; do
    VT_LIB_PATH=$lib python bench.py --no-cpu --simp-iters 0 --no-cfg5 --steps 50 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t apply', round(d['ms_per_step']*1e3,1),'us', round(d['value'],1),'GDOF/s frac', round(d['roofline']['frac'],3))"
  done
  VT_LIB_PATH=$lib python scripts/quick_apply.py 256 128 128 2>&1 | sed "s/^/$t /"
  VT_LIB_PATH=$lib python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py tests/test_gpu_solver.py -q -x -p no:cacheprovider -k "not cfg1" 2>&1 | tail -2 | sed "s/^/$t tests /"
done
