#!/bin/bash
# Runs ON the GPU box: compute-sanitizer memcheck / racecheck / synccheck over
# the small-config GPU suite (operator, V-cycle, PCG graph, Galerkin, slabs,
# design kernels).  Logs -> gpurun_out/sanitize_<tool>.log
#   bash scripts/sanitize.sh [memcheck racecheck synccheck]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SMALL_SOLVER="mgcg_matches or jacobi_and_plain or pcg_breakdown or design_kernels or graph_not_reused or small_trajectory or oc_infeasible"
SMALL_SLABS="apply_matches or vcycle_matches or mgcg_matches or nccl_transport or filter_bit or design_loop_matches"
tools=${*:-memcheck racecheck synccheck}
for tool in $tools; do
  log=gpurun_out/sanitize_${tool}.log
  : > $log
  if [ $tool = memcheck ]; then
    sets=("tests/test_gpu_operator.py" "tests/test_gpu_solver.py -k \"$SMALL_SOLVER\""
          "tests/test_gpu_galerkin.py -k \"levels or mgcg\"" "tests/test_gpu_slabs.py -k \"$SMALL_SLABS\""
          "tests/test_gpu_two_material.py -k \"sensitivities or rejects\""
          "tests/test_gpu_tail.py -k \"matches_multikernel or coarsest\"")
    extra="--leak-check full"
  else
    # shared-memory hazard / barrier checks: the TMA-ring operator, transfers,
    # V-cycle, coarse solve, PCG graph and the slab exchange at small sizes
    sets=("tests/test_gpu_operator.py -k \"tile_edges or multigrid_matches or vcycle_linear\""
          "tests/test_gpu_solver.py -k \"mgcg_matches or design_kernels\""
          "tests/test_gpu_galerkin.py -k \"levels\"" "tests/test_gpu_slabs.py -k \"apply_matches or filter_bit\""
          "tests/test_gpu_tail.py -k \"matches_multikernel\"")
    extra=""
  fi
  for s in "${sets[@]}"; do
    echo "=== $tool: $s" >> $log
    eval timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 20 \
      python -m pytest $s -x -q -p no:cacheprovider >> $log 2>&1
    echo "=== rc=$?" >> $log
  done
  grep -E "ERROR SUMMARY|=== |passed|failed" $log | tail -30
done
