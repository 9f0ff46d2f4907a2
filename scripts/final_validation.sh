#!/bin/bash
# Runs ON the GPU box: the end-of-round evidence in one call -- GPU test suite,
# smoke, bench (both arms), the bench's ncu launch list, ncu --set full of the
# graded apply and of the level-0 residual / smoother+dot, the per-kernel table
# of one MGPCG iteration.  Outputs under gpurun_out/<tag>_*.
#   bash scripts/final_validation.sh r2v3
cd "${GRAFT_REPO_ROOT:-/root/repo}"
T=${1:-final}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${T}_gputests.log 2>&1; tail -3 $O/${T}_gputests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; tail -c 400 $O/${T}_bench.json; echo
python bench.py --impl reference > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err; tail -c 300 $O/${T}_bench_ref.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches.csv \
    python bench.py --steps 2 --warmup 3 --simp-iters 0 --no-cfg5 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:hex8_tile_kernel -s 3 -c 1 -f -o $O/${T}_hex8 \
    python scripts/ncu_apply.py > /dev/null 2>&1
# level-0 smoother + r.z (hex8<SMOOTH, dot>) and residual (hex8<RESID>) of the PCG graph
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:hex8_tile_kernelILi2ELb1ELb0E -s 2 -c 1 -f -o $O/${T}_smooth python scripts/pcg_profile.py homogenized > $O/${T}_smooth.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:hex8_tile_kernelILi1ELb0ELb0E -s 2 -c 1 -f -o $O/${T}_resid python scripts/pcg_profile.py homogenized > $O/${T}_resid.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_pcg_homog.csv \
    python scripts/pcg_profile.py homogenized > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_pcg_gal.csv \
    python scripts/pcg_profile.py galerkin > /dev/null 2>&1
ls -la $O | grep "$T"
