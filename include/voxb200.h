/*
 * voxb200.h -- C ABI of the B200-native MGPCG hot path of voxtop
 * (arXiv 2201.12931).  Implemented by paper_2201_12931_b200/libvoxb200.so
 * (sm_100a CUDA kernels + a C++ runtime).  No torch types cross this
 * boundary: device buffers are plain pointers, sizes are integers.
 *
 * The reference (/root/reference/pkg, package `voxtop` 0.1.0) is pure Python
 * and has no FFI; each entry point below replaces one Python function of the
 * reference hot path and cites it as  [ref: file:line]  (paths relative to
 * pkg/src/voxtop/).  INTEGRATION.md shows the ctypes binding.
 *
 * ---------------------------------------------------------------- layouts
 * Node vectors ("vt node layout") hold 3 doubles per node, components
 * interleaved exactly like the reference dof numbering 3*node+comp
 * [ref: grid.py:1-10], but rows are padded to an even node pitch (TMA needs
 * 16-byte row strides) and the slab of node planes carries one ghost plane
 * below and one above:
 *     index(p, j, i, c) = ((p * (ny+1) + j) * row_pitch + i) * 3 + c,
 *     p = k - k0 + 1 (k = global node plane, [k0, k1) = owned element layers).
 * vt_vec_len() gives the length; vt_vec_upload/download convert to and from
 * the reference's flat (n_dofs,) numpy order.  Pad entries and ghost planes
 * must hold zeros (they do if the buffer was produced by this library or
 * zero-initialised).
 * Element fields passed by users (densities, sensitivities) are plain
 * (n_elements,) arrays in the reference element order [ref: grid.py:75-82].
 *
 * ---------------------------------------------------------------- errors
 * Every function returns a vt_status.  On failure vt_last_error() returns a
 * message formatted like the reference's exception text; the Python layer
 * maps the code to the reference exception class [ref: errors.py:7-24].
 *
 * All compute calls are asynchronous on `stream` (a cudaStream_t, NULL =
 * legacy default) unless stated otherwise.  A handle is not thread safe.
 */
#ifndef VOXB200_H
#define VOXB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  VT_OK = 0,
  VT_EINVAL = 1,        /* ValueError: shape / argument problems            */
  VT_ECUDA = 2,         /* CUDA runtime or launch failure                     */
  VT_ESETUP = 3,        /* SetupError  [ref: multigrid.py:280-316]            */
  VT_EBREAKDOWN = 4,    /* SolverBreakdown [ref: solver.py:81-156, 183-187]   */
  VT_EVOLUME = 5,       /* VolumeInfeasible [ref: optimize.py:271-292]        */
  VT_ENUMERICAL = 6,    /* NumericalError                                     */
  VT_ENOMEM = 7,        /* device allocation failure                          */
  VT_EDENSITY = 8       /* ValueError "density outside [0, 1]" [ref: element.py:105-106] */
} vt_status;

const char *vt_last_error(void);
int vt_version(void);
/* Number of CUDA kernel launches issued by this library since load (the
 * bench reports it as gpu_launches). */
uint64_t vt_launch_count(void);
/* device-to-device byte copy on stream (helper for bindings without a CUDA runtime) */
vt_status vt_copy(void *dst, const void *src, int64_t bytes, void *stream);

/* ------------------------------------------------------------------ grid
 * A vt_grid is one structured hex8 grid on one device: geometry, material
 * constants (nu, h), the fixed-dof mask, and scratch (reduction partials,
 * TMA descriptor cache).  Replaces the static part of OperatorState
 * [ref: operator.py:108-151] and StructuredGrid [ref: grid.py:45-111].
 *
 * node_mask: host array of (nz+1)*(ny+1)*(nx+1) bytes, bit c set <=> dof
 * 3*node+c is fixed.  k0/k1: owned element layers of this rank's z-slab
 * (0, nz for a single GPU).
 */
typedef struct vt_grid vt_grid;

vt_status vt_grid_create(vt_grid **out, int nx, int ny, int nz, double h, double nu,
                         const uint8_t *node_mask, int k0, int k1, int device);
vt_status vt_grid_destroy(vt_grid *g);
int64_t vt_vec_len(const vt_grid *g);   /* doubles in a vt node-layout vector  */
int64_t vt_elem_len(const vt_grid *g);  /* doubles in a vt element-layout field */
int64_t vt_n_fixed(const vt_grid *g);   /* fixed dofs of this slab              */
/* Profiling aid: when enabled, every hex8 launch on g records per CTA
 * {start ns, end ns, smid, items<<32 | tile origin} (4 x uint64); host_out
 * (optional) receives the last launch's records for max_ctas CTAs. */
vt_status vt_debug_trace(vt_grid *g, int enable, uint64_t *host_out, int max_ctas);

/* host <-> device conversion between the reference order and vt layout.
 * host pointers may be pageable or pinned; these calls are async on stream. */
vt_status vt_vec_upload(const vt_grid *g, const double *host, double *dev, void *stream);
vt_status vt_vec_download(const vt_grid *g, const double *dev, double *host, void *stream);

/* scale = E * (kmin + rho^p (1 - kmin)) into vt element layout (ghost layer
 * and padding zero) [ref: operator.py:142, element.py:102-108].  rho is a
 * plain device array of n_elements doubles.  Fails with VT_EDENSITY when a
 * density lies outside [0, 1] (synchronises to report it). */
vt_status vt_scale_from_density(vt_grid *g, const double *rho, double p, double kmin,
                                double E, double *scale, void *stream);

/* ---------------------------------------------------------- operator
 * v = K(rho) u with identity on fixed dofs; u is projected to zero on fixed
 * dofs before the product [ref: operator.py:58-81, 154-165]. */
vt_status vt_apply(vt_grid *g, const double *scale, const double *u, double *v, void *stream);
/* Solver-internal apply: u must already be zero on fixed dofs (every CG /
 * multigrid vector is); skips the projection pass of vt_apply. */
vt_status vt_apply_projected(vt_grid *g, const double *scale, const double *u, double *v,
                             void *stream);
/* v = K(rho) u from HOST memory to HOST memory (reference (n_dofs,) order),
 * streamed in `nchunks` z-chunks so the H2D copy, the operator and the D2H
 * copy overlap [ref: operator.py:154-165]; fixed dofs keep u (identity).
 * Pinned host buffers give full PCIe bandwidth.  Blocking. */
vt_status vt_apply_host(vt_grid *g, const double *scale, const double *u_host, double *v_host,
                        int nchunks, void *stream);
/* d = diag K, 1 on fixed [ref: operator.py:84-105, 168-174] */
vt_status vt_diagonal(vt_grid *g, const double *scale, double *d, void *stream);
/* r = f - K u, zero on fixed [ref: operator.py:177-184] */
vt_status vt_residual(vt_grid *g, const double *scale, const double *u, const double *f,
                      double *r, void *stream);
/* out = x . y over this slab's owned dofs (deterministic order); blocking. */
vt_status vt_dot(vt_grid *g, const double *x, const double *y, double *out, void *stream);
/* numpy-rounded updates over a whole node vector [ref: solver.py:131-158]:
 * mode 0 y = y + a*x, mode 1 y = y - a*x, mode 2 y = x + a*y */
vt_status vt_axpy(vt_grid *g, int mode, double a, const double *x, double *y, void *stream);
/* dst = src with fixed dofs zeroed (dst may equal src) [ref: solver.py:99] */
vt_status vt_project(vt_grid *g, const double *src, double *dst, void *stream);
/* K (n x n, device, n = n_dofs) = the dense global stiffness with identity
 * rows / columns on fixed dofs, bit-identical to the reference's np.add.at
 * assembly [ref: operator.py:187-205]; scale: plain (n_elements,) device
 * array in the reference element order, k0: 576 device doubles.  The caller
 * enforces the reference's dense guard. */
vt_status vt_assemble_dense(vt_grid *g, const double *scale, const double *k0, double *K,
                            void *stream);

/* ---------------------------------------------------------- multigrid
 * Homogenized geometric multigrid [ref: multigrid.py:150-499].  Level 0 is
 * `fine`; levels are created by halving, coarse fixed dofs = fine fixed dofs
 * at even nodes [ref: multigrid.py:137-141]. */
typedef struct vt_hier vt_hier;

vt_status vt_hier_create(vt_hier **out, vt_grid *fine, int n_levels, double omega, int sweeps);
/* scheme 0: homogenized (coarse operators E s(mean rho) K0(2^l h), rebuilt on
 * the fly); scheme 1: galerkin, the reference default -- per-element 24x24
 * coarse matrices P^T K P with the fixed-dof projection [ref: multigrid.py:
 * 59-81, 216-278], stored on levels >= 1 (576 doubles per coarse element). */
vt_status vt_hier_create_ex(vt_hier **out, vt_grid *fine, int n_levels, double omega, int sweeps,
                            int scheme);
int vt_hier_scheme(const vt_hier *H);
/* Fused coarse tail: the V-cycle levels from the first one with at most
 * `nodes` nodes down to the coarsest direct solve and back up run as ONE
 * thread-block-cluster kernel (tail.cu) instead of ~7 launches per level.
 * Applies to hierarchies created afterwards; 0 disables.  Returns the previous
 * budget (default 0 = off, measured slower than the PDL kernel chain on B200;
 * or the VT_TAIL_NODES environment variable). */
long long vt_tail_config(long long nodes);
/* first level the fused tail covers in a V-cycle entered at level 0; -1: none */
int vt_hier_tail_level(vt_hier *H);
/* profiling: enable (1) / disable (0) a 64-slot device record of %globaltimer
 * after every phase of the fused tail (slot 63: kernel start); host_out (may be
 * NULL) receives max_slots slots after a device synchronize */
vt_status vt_tail_trace(int enable, uint64_t *host_out, int max_slots);
vt_status vt_hier_destroy(vt_hier *H);
int vt_hier_levels(const vt_hier *H);
vt_grid *vt_hier_grid(vt_hier *H, int level);
/* coarse element densities + scales + per-level diagonal + coarsest direct
 * factor [ref: multigrid.py:201-233, 280-316]; rho: plain fine densities,
 * scale0: fine scale in vt element layout. */
vt_status vt_hier_refresh(vt_hier *H, const double *rho, const double *scale0, double p,
                          double kmin, double E, void *stream);
/* z = V-cycle(f) [ref: multigrid.py:404-430] */
vt_status vt_hier_vcycle(vt_hier *H, const double *f, double *z, void *stream);
/* level-l building blocks (tests / API parity) */
vt_status vt_hier_restrict(vt_hier *H, int l, const double *fine, double *coarse, void *stream);
vt_status vt_hier_prolong(vt_hier *H, int l, const double *coarse, double *fine, void *stream);
vt_status vt_hier_jacobi(vt_hier *H, int l, const double *u, const double *f, int sweeps,
                         double *out, void *stream);
vt_status vt_hier_level_apply(vt_hier *H, int l, const double *u, double *v, void *stream);
vt_status vt_hier_level_diag(vt_hier *H, int l, double *d, void *stream);
vt_status vt_hier_coarse_solve(vt_hier *H, const double *f, double *u, void *stream);
/* device pointer to level-l element scale / plain density (vt layouts) */
const double *vt_hier_level_scale(vt_hier *H, int l);
/* galerkin: level-l element matrices (n_elements_l x 576, reference element
 * order, row-major 24x24); NULL for homogenized hierarchies or l = 0.  The
 * solver stores the symmetric matrices as their packed upper triangle (300
 * doubles per element); this call expands them into a hierarchy-owned buffer
 * that stays valid until the next call (synchronizes the device). */
const double *vt_hier_level_mats(vt_hier *H, int l);
const double *vt_hier_level_rho(vt_hier *H, int l);

/* ---------------------------------------------------------- solver
 * Preconditioned CG with the reference recurrences, true residual every 50
 * iterations and on convergence, and identical breakdown checks
 * [ref: solver.py:62-167]; precond: 0 none, 1 Jacobi [ref: solver.py:57-59],
 * 2 multigrid V-cycle (H required) [ref: solver.py:170-191].
 * x: in = warm start (ignored unless warm), out = solution.  Blocking. */
typedef struct {
  int iterations;
  double final_rel_residual;
  int precond_applications;
  int converged;
  double residual_drift;
  int breakdown;          /* 0 none; 1 rz<=0 (it 0 or k); 2 non-finite pq; 3 pq<=0; 4 non-finite residual; 5 non-finite rhs */
  int breakdown_iter;
  double breakdown_value;
} vt_solve_report;

vt_status vt_pcg(vt_grid *g, const double *scale, int precond, vt_hier *H, const double *f,
                 double *x, int warm, double tol, int max_iterations, vt_solve_report *rep,
                 void *stream);

/* ---------------------------------------------------------- design loop
 * [ref: optimize.py:186-302] */
/* c = f . u (blocking) */
vt_status vt_compliance(vt_grid *g, const double *f, const double *u, double *c, void *stream);
/* dc_e = -E s'(rho_e) u_e'K0 u_e (+ 2 u_e.g_unit when grav_axis >= 0), plain
 * element order [ref: optimize.py:195-213]; grav_coef = -uw*g*h^3/8 */
vt_status vt_sensitivities(vt_grid *g, const double *u, const double *rho, double p, double kmin,
                           double E, int grav_axis, double grav_coef, double *dc, void *stream);
/* Two-material SIMP (BASELINE cfg4; NO reference counterpart -- the
 * reference's SPEC.md:15,178 lists multi-material as never developed, so this
 * extends simp_scale / sensitivities [ref: element.py:102-118,
 * optimize.py:195-213] and is pinned only through its single-material limit
 * eB = 1 and finite differences).  Element modulus E s(rho) m(phi) with
 * m = eB + (1 - eB) phi^p, eB = E_B / E_A in [0, 1].
 * scale: vt element layout; rho_mg (optional, plain element order) =
 * rho m^(1/p), the density the homogenized coarse levels average.
 * VT_EDENSITY when rho or phi lies outside [0, 1]. */
vt_status vt_scale_two_material(vt_grid *g, const double *rho, const double *phi, double p,
                                double kmin, double E, double eB, double *scale, double *rho_mg,
                                void *stream);
/* dc_rho = -E s'(rho) m(phi) u_e'K0u_e (+ gravity term as vt_sensitivities),
 * dc_phi = -E s(rho) p phi^(p-1) (1 - eB) u_e'K0u_e */
vt_status vt_sensitivities_two_material(vt_grid *g, const double *u, const double *rho,
                                        const double *phi, double p, double kmin, double E,
                                        double eB, int grav_axis, double grav_coef, double *dc_rho,
                                        double *dc_phi, void *stream);
/* f = scatter(rho_e g_unit) (+ f_ext) (zero on fixed if zero_fixed)
 * [ref: optimize.py:216-231] */
vt_status vt_gravity_load(vt_grid *g, const double *rho, int grav_axis, double grav_coef,
                          const double *f_ext, int zero_fixed, double *f, void *stream);
/* sensitivity filter with a (2R+1)^3 kernel in (dk,dj,di) order; wsum is
 * computed on the device at creation [ref: optimize.py:110-179] */
typedef struct vt_filter vt_filter;
vt_status vt_filter_create(vt_filter **out, vt_grid *g, int R, const double *kernel_host);
vt_status vt_filter_destroy(vt_filter *F);
const double *vt_filter_wsum(vt_filter *F);
vt_status vt_filter_apply(vt_filter *F, const double *dc, const double *rho, double gamma,
                          double *dcf, void *stream);
/* out = correlate(field, kernel), zero padding [ref: optimize.py:139-144] */
vt_status vt_filter_correlate(vt_filter *F, const double *field, double *out, void *stream);
/* OC update with bisected multiplier [ref: optimize.py:245-302]; classes:
 * int8 per element (0 active).  Blocking; VT_EVOLUME on infeasibility. */
vt_status vt_oc_update(vt_grid *g, const double *rho, const int8_t *classes, const double *dc,
                       const double *dv, double volfrac, double move, double eta, double q,
                       double *rho_out, double *lam, int *steps, void *stream);
/* The same OC update on plain (nel,) device arrays with no grid handle (the
 * public oc_update of a bare density field) [ref: optimize.py:245-302]. */
vt_status vt_oc_update_flat(long long nel, const double *rho, const int8_t *classes, const double *dc,
                            const double *dv, double volfrac, double move, double eta, double q,
                            double *rho_out, double *lam, int *steps, void *stream);
/* max |a-b| and mean of a over active elements (blocking helpers of run()) */
vt_status vt_change_volume(vt_grid *g, const double *a, const double *b, const int8_t *classes,
                           double *max_abs_diff, double *active_mean, void *stream);

/* ---------------------------------------------------------- z-slab decomposition
 * The MGPCG solve across ranks (the reference is single-process,
 * so these entry points have no reference counterpart -- they distribute
 * vt_apply / vt_hier_* / vt_pcg above).  Rank g owns element layers
 * [kbounds[g], kbounds[g+1]) of the fine grid; kbounds are multiples of
 * 2^dist_level, levels 0..dist_level are slab-distributed and the coarse tail
 * (dist_level+1 .. levels-1, incl. the coarsest direct solve) is replicated.
 * nccl_id == NULL: all nranks slabs live in this process on `device` and
 * exchange through device copies (nlocal == nranks); otherwise one slab per
 * process (nlocal == 1, rank0 = this rank) and NCCL (dlopen'ed, VT_NCCL_LIB)
 * carries the halos and the rank-ordered dot products.  Slab vectors use the
 * vt node layout of vt_dist_grid(D, i, 0) (ghost planes included).  Pointer
 * arrays (`double *const *`) hold one device pointer per local slab. */
typedef struct vt_dist vt_dist;

int vt_nccl_id_bytes(void);
vt_status vt_nccl_unique_id(uint8_t *out, int nbytes);
vt_status vt_dist_create(vt_dist **out, int nx, int ny, int nz, double h, double nu,
                         const uint8_t *node_mask, int levels, double omega, int nranks,
                         int rank0, int nlocal, const int *kbounds, int dist_level,
                         const uint8_t *nccl_id, int device);
/* One slab per process with the peer-memory transport (csrc/peer.cu): every
 * exchange is one kernel that loads the neighbours' staged planes straight
 * from their device memory (CUDA IPC; NVLink / NVSwitch across the GPUs of a
 * box, the same HBM when ranks share a GPU).  After creation every rank
 * exports vt_dist_peer_handle, the handles are all-gathered (rank order) and
 * passed to vt_dist_peer_open before the first exchange. */
vt_status vt_dist_create_peer(vt_dist **out, int nx, int ny, int nz, double h, double nu,
                              const uint8_t *node_mask, int levels, double omega, int nranks,
                              int rank, const int *kbounds, int dist_level, int device);
int vt_peer_handle_bytes(void);
vt_status vt_dist_peer_handle(vt_dist *D, uint8_t *out, int nbytes);
vt_status vt_dist_peer_open(vt_dist *D, const uint8_t *handles, int nbytes);
vt_status vt_dist_destroy(vt_dist *D);
/* Switch to the reference's default Galerkin scheme [ref: multigrid.py:216-278]
 * before the first refresh (dist_level must be 1): levels 0 and 1 stay on the
 * slabs (level 1 matrix-free through the fine kernels), the stored-matrix
 * levels >= 2 and the coarsest solve run replicated, built each refresh from
 * the gathered fine scale field (csrc/dist_galerkin.cu). */
vt_status vt_dist_set_scheme(vt_dist *D, int scheme);
int vt_dist_scheme(const vt_dist *D);
int vt_dist_levels(const vt_dist *D);
int vt_dist_dist_level(const vt_dist *D);
int vt_dist_nlocal(const vt_dist *D);
vt_grid *vt_dist_grid(vt_dist *D, int slab, int level);
vt_hier *vt_dist_tail(vt_dist *D);
uint64_t vt_dist_graph_nodes(const vt_dist *D);
/* level-0 element scales of the local slabs; exchanges the ghost layer */
vt_status vt_dist_set_scale(vt_dist *D, const double *const *scale0, void *stream);
/* coarse levels + replicated tail + coarsest factor [ref: multigrid.py:201-233]; blocking */
vt_status vt_dist_refresh(vt_dist *D, const double *const *rho, const double *const *scale0,
                          double p, double kmin, double E, void *stream);
/* v = K u per slab (u zero on fixed dofs; its ghost planes are refreshed) */
vt_status vt_dist_apply(vt_dist *D, double *const *u, double *const *v, void *stream);
vt_status vt_dist_dot(vt_dist *D, const double *const *x, const double *const *y, double *out,
                      void *stream);
vt_status vt_dist_vcycle(vt_dist *D, const double *const *f, double *const *z, void *stream);
/* MGPCG over all ranks, same recurrences as vt_pcg [ref: solver.py:62-191]; blocking */
vt_status vt_dist_pcg(vt_dist *D, const double *const *f, double *const *x, int warm, double tol,
                      int max_iterations, vt_solve_report *rep, void *stream);
/* design step on the slabs [ref: optimize.py:139-302]: element fields are the
 * plain slab ranges of the reference element order (slab i: layers
 * [kbounds[rank], kbounds[rank+1])).  Sensitivities refresh u's ghost planes;
 * the filter exchanges R element layers of rho*dc with each neighbour and is
 * bit-identical to the single-GPU filter; OC bisection and change/volume sum
 * per rank, all-gather and add in rank order (identical decisions on every
 * rank).  oc_update / change_volume are blocking. */
vt_status vt_dist_sensitivities(vt_dist *D, double *const *u, const double *const *rho, double p,
                                double kmin, double E, int grav_axis, double grav_coef,
                                double *const *dc, void *stream);
/* self-weight load f = scatter(rho_e g_unit) (+ f_ext), zero on fixed if
 * zero_fixed [ref: optimize.py:216-231]; exchanges the element layer below */
vt_status vt_dist_gravity_load(vt_dist *D, const double *const *rho, int grav_axis, double grav_coef,
                               const double *const *f_ext, int zero_fixed, double *const *f,
                               void *stream);
vt_status vt_dist_sensitivities_two_material(vt_dist *D, double *const *u, const double *const *rho,
                                             const double *const *phi, double p, double kmin, double E,
                                             double e_ratio, int grav_axis, double grav_coef,
                                             double *const *dc_rho, double *const *dc_phi, void *stream);
vt_status vt_dist_filter_create(vt_dist *D, int R, const double *kernel_host);
vt_status vt_dist_filter_apply(vt_dist *D, const double *const *dc, const double *const *rho,
                               double gamma, double *const *dcf, void *stream);
vt_status vt_dist_oc_update(vt_dist *D, const double *const *rho, const int8_t *const *classes,
                            const double *const *dc, const double *const *dv, double volfrac,
                            double move, double eta, double q, double *const *rho_out,
                            double *lam, int *steps, void *stream);
vt_status vt_dist_change_volume(vt_dist *D, const double *const *a, const double *const *b,
                                const int8_t *const *classes, double *max_abs_diff,
                                double *active_mean, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* VOXB200_H */
