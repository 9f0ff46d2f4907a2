#!/bin/bash
# Runs ON the GPU box: A/B of library variants (tags of _build.py; "base" = the
# default libvoxb200.so) on the solve path: ms per MGPCG iteration at cfg2 for
# both schemes, run twice, interleaved, plus the transfer / V-cycle parity tests.
#   bash scripts/ab_solve.sh base prb4 prb6
cd "${GRAFT_REPO_ROOT:-/root/repo}"
lib_of() { if [ "$1" = base ]; then echo $PWD/paper_2201_12931_b200/libvoxb200.so; else echo $PWD/paper_2201_12931_b200/libvoxb200_$1.so; fi; }
for rep in 1 2; do
  for t in "$@"; do
    VT_LIB_PATH=$(lib_of $t) python scripts/pcg_time.py 2>&1 | sed "s/^/$t /"
  done
done
for t in "$@"; do
  VT_LIB_PATH=$(lib_of $t) python -m pytest tests/test_gpu_operator.py tests/test_gpu_galerkin.py -q -x -p no:cacheprovider \
    -k "transfers or multigrid or vcycle or galerkin" 2>&1 | tail -1 | sed "s/^/$t tests /"
done
