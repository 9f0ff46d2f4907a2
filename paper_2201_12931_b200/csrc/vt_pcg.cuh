// Device-resident PCG control block and launchers (see vectors.cu, runtime.cu).
#pragma once
#include "vt_internal.h"

namespace vt {

// Lives in device memory; scalar kernels update it, every vector kernel of
// an iteration reads its skip words so the host never blocks inside an
// iteration.  Mirrors the local variables of the reference pcg()
// [ref: solver.py:62-167].
struct PcgCtl {
  int stop;         // solve finished (converged or breakdown): all kernels skip
  int skip_rec;     // skip the recursive r -= alpha q update (k % 50 == 0)
  int skip_true50;  // skip the periodic true residual (k % 50 != 0)
  int skip_cand;    // skip the convergence-candidate true residual
  int skip_swap;    // skip copying the candidate residual into r
  int converged;
  int k;
  int err, err_iter;
  int precond_apps;
  int skip_xc;      // skip the candidate's x update (no candidate, or x already current)
  int x_done;       // x already holds x + alpha p this iteration (xpby must not add it)
  double err_val;
  double rz, pq, alpha, beta, rel, fnorm, tol, drift;
};

vt_status launch_pcg_update(vt_grid* G, PcgCtl* ctl, double* x, const double* p, double* r,
                            const double* q, double* partial, int with_r, cudaStream_t s,
                            const double* w = nullptr, double* u0 = nullptr);
// x == nullptr: p = z + beta p only; else also x += alpha p (old p) unless
// ctl->x_done -- the x update deferred from pcg_update (one stream fewer)
vt_status launch_pcg_xpby(vt_grid* G, PcgCtl* ctl, const double* z, double* p, cudaStream_t s,
                          double* x = nullptr);
vt_status launch_copy(vt_grid* G, const int* skip, const double* src, double* dst,
                      cudaStream_t s, int grid = 0);
vt_status launch_jacobi_precond(vt_grid* G, const int* stop, const double* r, const double* d,
                                double* z, double* partial, cudaStream_t s);
vt_status launch_pcg_s1(PcgCtl* c, const double* partial, int n, cudaStream_t s);
vt_status launch_pcg_s2(PcgCtl* c, const double* partial, int n_rec, int n_true,
                        cudaStream_t s);
vt_status launch_pcg_s3(PcgCtl* c, const double* partial, int n, cudaStream_t s);
vt_status launch_pcg_s4(PcgCtl* c, const double* partial, int n, int counts, cudaStream_t s);
vt_status launch_jacobi0(vt_grid* G, const double* scale, double omega, const double* f,
                         double* u, const int* stop, cudaStream_t s);
vt_status launch_wdiag(vt_grid* G, const double* scale, double omega, double* w, cudaStream_t s);
vt_status launch_jacobi0w(vt_grid* G, const double* w, const double* f, double* u, const int* stop,
                          cudaStream_t s, const PcgCtl* fused = nullptr);

}  // namespace vt
