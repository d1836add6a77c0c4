/*
 * msb.h — C ABI of libmsb, the B200 (sm_100a) hot path of the iterative
 * multiscale restriction-smoothed-basis (MsRSB) pressure solver of
 * Klemetsdal, Møyner & Lie, arXiv 2001.01624 ("PAPER.md").
 *
 * Calls follow BASELINE.json north_star's problem statement:
 *   build_tpfa(grid, K, wells)        -> msb_build_tpfa
 *   build_partition / build_support   -> msb_partition_cartesian, msb_level_create_cartesian,
 *                                        msb_level_create_split; NEXT-3: msb_partition_wells,
 *                                        msb_partition_indicator, msb_level_create_general
 *   smooth_basis(P, iters, w)         -> msb_smooth_basis
 *   coarse_assemble(R, A, P) -> A_c   -> msb_coarse_assemble
 *   add_dynamic_basis(dp)             -> msb_add_dynamic_basis
 *   ms_iterate(b, tol)                -> msb_ms_iterate
 * Every arithmetic step runs in CUDA kernels of this library; the library has no
 * CPU fallback (a missing device is MSB_ECUDA).
 *
 * Conventions (all calls):
 *  - Status: 0 MSB_OK; >0 warning with valid outputs; <0 error.  msb_last_error()
 *    returns a thread-safe-per-context message, valid until the next call on that context.
 *  - Ownership: handles (msb_op, msb_level, msb_solver) own device arrays obtained
 *    through the context allocator and free them in *_destroy.  Caller arrays are
 *    never retained past the call that receives them.
 *  - Pointers: arguments documented "host|dev" may be host memory (pageable or pinned)
 *    or device memory of the context's device; the library detects which and stages
 *    host data through device buffers (copies enqueued on the context stream).
 *    Arguments documented "dev" must be device memory.
 *  - Streams: all work is enqueued on the context stream.  Calls that return host
 *    scalars (counts, iteration numbers, norms) synchronise that stream.
 *  - Layout: fp64 values, int32 cell/block indices, natural cell order
 *    c = i + nx*(j + ny*k).  Per-axis face arrays are compact:
 *      x-faces f = i + (nx-1)*(j + ny*k), y-faces f = i + nx*(j + (ny-1)*k),
 *      z-faces f = i + nx*(j + ny*k)   (left/lower cell of the face).
 */
#ifndef MSB_H
#define MSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t msb_status;
enum {
  MSB_OK = 0,
  MSB_NOT_CONVERGED = 1,   /* warning: max_iter / max_sweeps reached; outputs valid   */
  MSB_EINVAL = -1,         /* null handle/pointer, bad size or argument               */
  MSB_EDIM = -2,           /* dimension mismatch                                       */
  MSB_EZERO_DIAG = -3,     /* zero diagonal in A_T                       */
  MSB_ESINGULAR = -4,      /* coarse pivot <= 1e-14 * max|A_c|            */
  MSB_EINCONSISTENT = -5,  /* A singular: sealing faces (T = 0) cut off a compartment
                              without the gauge cell 0, so the A_00 gauge (reading A7)
                              does not fix its pure-Neumann null space      */
  MSB_EDIVERGED = -6,      /* residual > 1e6 * initial residual           */
  MSB_ENOMEM = -7,         /* allocator returned NULL                                  */
  MSB_ECUDA = -8           /* CUDA runtime error / no device                           */
};

typedef struct msb_ctx_s* msb_ctx;
typedef struct msb_op_s* msb_op;
typedef struct msb_level_s* msb_level;
typedef struct msb_solver_s* msb_solver;

/* Structured grid of nx*ny*nz cells with sizes dx, dy, dz. */
typedef struct {
  int32_t nx, ny, nz;
  double dx, dy, dz;
} msb_grid;

/* Source/sink cell (well as source term): rate > 0 injection. */
typedef struct {
  int32_t cell;
  double rate;
} msb_source;

/* Allocator hook: returns device memory of `bytes` on the context device, or NULL. */
typedef void* (*msb_alloc_fn)(size_t bytes, void* user);
typedef void (*msb_free_fn)(void* ptr, void* user);

/* ---------------------------------------------------------------- context */

/* Create a context on `device` that enqueues on `cuda_stream` (a cudaStream_t; NULL =
 * legacy default stream).  alloc/free may be NULL (then cudaMalloc/cudaFree). */
msb_status msb_ctx_create(msb_ctx* out, int device, void* cuda_stream, msb_alloc_fn alloc,
                          msb_free_fn free_fn, void* user);
msb_status msb_ctx_destroy(msb_ctx ctx);
msb_status msb_ctx_set_stream(msb_ctx ctx, void* cuda_stream);
const char* msb_last_error(msb_ctx ctx);
/* Library version string and the number of this library's kernel launches so far
 * (all contexts); used by the bench to report "gpu_launches". */
const char* msb_version(void);
int64_t msb_launch_count(void);

/* ---------------------------------------------------------------- TPFA (row a1)
 * PAPER.md:101 two-point flux; SPEC.md:159-167:
 *   t_{i,a} = K_{i,a} A_a / (Δ_a/2),  T_f = (1/t_i + 1/t_l)^{-1} * mult_f * mob_f.
 * A_T = Σ_f T_f (e_i - e_l)(e_i - e_l)^T (zero row sums; used to smooth the basis,
 * reading A2); the solve matrix A doubles A_00 (pure-Neumann gauge, reading A7).
 * K      host|dev, 3N doubles, SoA kx | ky | kz, all > 0 (else MSB_EINVAL).
 * mult   host|dev or NULL: three compact face arrays concatenated (x | y | z faces).
 * mob    host|dev or NULL: same layout, face mobility λ_f (config 4).
 * src    host array of n_src sources; q_i = Σ rates of sources in cell i.
 * out    new operator; owns T face arrays (cell-padded), q and a face-open mask
 *        (mult == 1) used by the fault-split partition.
 * Errors: MSB_EINVAL as above; MSB_EDIM when 3N >= 2^31 (cells are int32-indexed). */
msb_status msb_build_tpfa(msb_ctx ctx, const msb_grid* grid, const double* K, const double* mult,
                          const double* mob, const msb_source* src, int32_t n_src, msb_op* out);
/* Replace the face mobility (host|dev, compact face layout) and rebuild T. */
msb_status msb_op_set_mobility(msb_ctx ctx, msb_op op, const double* mob);
/* Copy out T (three compact face arrays, x|y|z, host|dev) and/or q (N, host|dev); NULL skips. */
msb_status msb_op_export(msb_ctx ctx, msb_op op, double* T_faces, double* q);
/* y = A x (gauge included) for device vectors of length N (diagnostics / tests). */
msb_status msb_op_apply(msb_ctx ctx, msb_op op, const double* x_dev, double* y_dev);
msb_status msb_op_destroy(msb_op op);

/* ---------------------------------------------------------------- partitions / supports (row a2)
 * Cartesian partition: block (floor(x/bx), floor(y/by), floor(z/bz)),
 * natural block order; the last block along an axis may be ragged.
 * part  host|dev int32[N] output (may be NULL); M_out host int32. */
msb_status msb_partition_cartesian(msb_ctx ctx, const msb_grid* grid, int32_t bx, int32_t by,
                                   int32_t bz, int32_t* part, int32_t* M_out);

/* Level over the Cartesian partition with open-box supports (reading A3): cell x lies
 * in S_J along axis a iff C(J-1) < 2x+1 < C(J+1), C(J) = lo_J + hi_J (doubled block
 * centre), the limit dropped at the domain boundary.  P := indicator (P^0).
 * Stored as 8 parity slot planes (slot bit a = block index parity along axis a).
 * nnz_out host, may be NULL. */
msb_status msb_level_create_cartesian(msb_ctx ctx, msb_op op, int32_t bx, int32_t by, int32_t bz,
                                      msb_level* out, int64_t* nnz_out);
/* Fault-split level (readings A4, A20): blocks = connected components
 * of each parent Cartesian block over faces with multiplier == 1, numbered by ascending
 * minimum cell; supports = flood fill from each block inside the parent's support box
 * across faces with multiplier == 1.  Explicit ELL pattern, columns ascending. */
msb_status msb_level_create_split(msb_ctx ctx, msb_op op, msb_level parent, msb_level* out,
                                  int64_t* nnz_out);
/* Level with a caller-supplied partition and constant basis P_ij = [part_i == j]
 * (PAPER.md:260 caption).  part host|dev int32[N], values in [0, M). */
msb_status msb_level_create_constant(msb_ctx ctx, msb_op op, const int32_t* part, int32_t M,
                                     msb_level* out);
/* ---------------------------------------------------------------- static partitions (§8 NEXT-3)
 * Well partition ("one for each well plus one to ensure partition of unity";
 * SPEC.md:410-416; reading B9): well w owns the cells whose Chebyshev index distance to its
 * nearest perforation is <= radius (a cell in reach of several wells joins the nearest,
 * ties to the lower well index); block n_wells holds every other cell and is omitted when
 * empty.  perf_ptr host int32[n_wells+1] (CSR offsets into perf_cells), perf_cells host
 * int32[perf_ptr[n_wells]] cell indices; part host|dev int32[N] out; M_out host.
 * Errors: MSB_EINVAL for radius < 0, a well without perforations or a cell outside the grid. */
msb_status msb_partition_wells(msb_ctx ctx, const msb_grid* grid, const int32_t* perf_ptr,
                               const int32_t* perf_cells, int32_t n_wells, int32_t radius,
                               int32_t* part, int32_t* M_out);
/* Indicator partition ("agglomerates cells into coarse blocks based on a
 * flow indicator"; reading B10): bin_i = #{e : edges[e] <= |ind_i|}
 * (absolute edges, strictly increasing, n_edges <= 8), connected components of equal bins
 * over the grid faces, components below s_min merged into one block per bin with s_min
 * doubling from 1 until at most max_blocks blocks remain (the dynamic stage's rule, A15);
 * numbered by ascending minimum cell.  ind host|dev double[N]; part host|dev int32[N] out. */
msb_status msb_partition_indicator(msb_ctx ctx, msb_op op, const double* ind, const double* edges,
                                   int32_t n_edges, int32_t max_blocks, int32_t* part,
                                   int32_t* M_out);
/* Level on a general partition (§8 NEXT-3; reading B8): supports
 * S_j = block j dilated by `halo` layers of the graph of A_T (faces with base T > 0),
 * explicit ELL pattern with ascending columns (at most 16 per cell, else MSB_EINVAL),
 * P := constant basis of the partition (P^0), ready for msb_smooth_basis (halo 0: the
 * constant-basis level).  part host|dev int32[N], values in [0, M). */
msb_status msb_level_create_general(msb_ctx ctx, msb_op op, const int32_t* part, int32_t M,
                                    int32_t halo, msb_level* out, int64_t* nnz_out);
/* Level facts: M, nnz, slot width W (planes), and the partition (host|dev int32[N], may be NULL). */
msb_status msb_level_info(msb_ctx ctx, msb_level lev, int32_t* M, int64_t* nnz, int32_t* W,
                          int32_t* part);
/* Parity dump of P as CSR with ascending columns: rowptr int64[N+1], cols int32[nnz],
 * vals double[nnz] (each host|dev, any may be NULL), and A_c dense M*M row-major
 * (host|dev, NULL skips; requires a dense coarse operator). */
msb_status msb_level_export(msb_ctx ctx, msb_level lev, int64_t* rowptr, int32_t* cols,
                            double* vals, double* Ac_dense);
/* Overwrite P from CSR (same pattern as exported; host|dev) — lockstep tests.  Imported
 * rows need not sum to one: the level's next msb_coarse_assemble accumulates every entry
 * of A_c (until a msb_smooth_basis call renormalises the rows again). */
msb_status msb_level_import_values(msb_ctx ctx, msb_level lev, const double* vals);
/* Parity dump of a Cartesian level's assembled A_c in its box-stencil storage, as COO in
 * row-major order (every in-range slot (a, b), |b - a| <= 2 blocks per axis, zeros
 * included): nnz_out host; rows, cols int32[nnz] and vals double[nnz] (host|dev, each may
 * be NULL: call once with NULLs for nnz).  Available for every Cartesian level (the dense
 * dump of msb_level_export only where the dense solver is used, M <= 4096).
 * Errors: MSB_EINVAL for an explicit level or before msb_coarse_assemble. */
msb_status msb_level_export_coarse(msb_ctx ctx, msb_level lev, int64_t* nnz_out, int32_t* rows,
                                   int32_t* cols, double* vals);
msb_status msb_level_destroy(msb_level lev);

/* ---------------------------------------------------------------- basis smoothing (row a3)
 * Restricted damped-Jacobi sweeps (BASELINE.json north_star; SPEC.md:428-436;
 * readings A2, A5, A6, A16), positive form on the fixed pattern:
 *   P^_ij = (1-ω) P_ij + (ω/D_i) Σ_{l~i} T_il P_lj,   P_ij <- P^_ij / Σ_k P^_ik  (every row),
 *   δ_n = max |P^{n+1} - P^n|.
 * Stops after sweep n when δ_n <= tol (tol < 0: never) or n = max_sweeps.
 * Returns MSB_NOT_CONVERGED if max_sweeps was reached with tol >= 0 and δ > tol.
 * deltas: host array of max_sweeps doubles or NULL (δ history). */
msb_status msb_smooth_basis(msb_ctx ctx, msb_level lev, msb_op op, int32_t max_sweeps,
                            double omega, double tol, int32_t* sweeps_done, double* last_delta,
                            double* deltas);

/* ---------------------------------------------------------------- Galerkin coarse operator (rows a4, a5)
 * A_c = P^T A P (R = P^T) accumulated face by face:
 *   A_c = Σ_f T_f (P_i. - P_l.)^T (P_i. - P_l.) + A_00^T (P_0.)^T P_0.  (gauge term),
 * then factorised on the device (SPD Cholesky = LU without pivoting for SPD A_c,
 * PAPER.md:410) and, for dense A_c, inverted so that each coarse solve is one GEMV.
 * For M <= 8192 the sum is exact in 128-bit fixed point (run-to-run identical); when the
 * rows of P sum to one (created or smoothed levels: MsRSB's partition of unity) each face
 * adds only the lower off-diagonal products and the diagonal is minus the row's
 * off-diagonal total plus the gauge term — the same matrix up to the rounding of P's row
 * sums.  Returns MSB_ESINGULAR if a pivot is <= 1e-14 * max|A_c|, MSB_EINCONSISTENT when
 * the faces with T > 0 leave a compartment without the gauge cell 0 (A, hence A_c, is
 * then singular). */
msb_status msb_coarse_assemble(msb_ctx ctx, msb_level lev, msb_op op);

/* ---------------------------------------------------------------- solver (rows a6–a11)
 * Multibasis Richardson iteration, Eq. (8): for each level ℓ in order,
 *   pre  (post_smooth = 0): ν damped-Jacobi sweeps x <- x + ω_s D_A^{-1}(b - A x), then
 *                            x <- x + P (A_c)^{-1} P^T (b - A x);
 *   post (post_smooth = 1): the coarse correction first, then the ν sweeps.
 * Dynamic stage (dyn_enable; readings A12, A14, A15): from
 * iteration k >= 2, Δp = x_start(k) - x_start(k-1) is binned at dyn_edge{0,1}*max|Δp|,
 * split into connected components (canonical numbering by minimum cell), small
 * components merged per bin until at most dyn_max_blocks blocks, and appended as a
 * constant-basis stage.  Levels must have been assembled (msb_coarse_assemble).
 * Errors: MSB_EINCONSISTENT when the faces with T > 0 do not connect every cell to the
 * gauge cell 0 (A is then singular: "pre: A nonsingular"); MSB_EDIM for a level
 * of another grid; MSB_EINVAL for an unassembled level. */
msb_status msb_solver_create(msb_ctx ctx, msb_op op, const msb_level* levels, int32_t n_levels,
                             double omega_s, int32_t nu, int32_t post_smooth, int32_t dyn_enable,
                             double dyn_edge0, double dyn_edge1, int32_t dyn_max_blocks,
                             msb_solver* out);
/* Build the dynamic constant-basis stage from a caller Δp (host|dev, N doubles) and
 * install it as the solver's current dynamic stage.  M_dyn_out host; part_out host|dev
 * int32[N] or NULL.  M_dyn = 0 (stage cleared) when max|Δp| = 0. */
msb_status msb_add_dynamic_basis(msb_ctx ctx, msb_solver s, const double* dp, int32_t* M_dyn_out,
                                 int32_t* part_out);
/* Richardson iteration from x0 (x: host|dev, in x0 / out x) for right-hand side b
 * (host|dev; NULL = the operator's q).  Stops when ||b - A x||_2 <= tol ||b||_2 after a
 * full cycle, or at max_iter (MSB_NOT_CONVERGED); fixed_iters > 0 runs exactly that
 * many cycles.  res_hist: host array of (max(max_iter, fixed_iters) + 1) doubles or
 * NULL (ρ_0..ρ_k).  dyn_M_hist: host int32 array (same length) or NULL: M_dyn used in
 * each iteration (0 = no dynamic stage). */
msb_status msb_ms_iterate(msb_ctx ctx, msb_solver s, const double* b, double* x, double tol,
                          int32_t max_iter, int32_t fixed_iters, int32_t* iters_out,
                          double* res_hist, int32_t* dyn_M_hist);
msb_status msb_solver_destroy(msb_solver s);
/* Stage smoother (§8 NEXT-2): kind 0 = damped Jacobi with the solver's omega_s (reading A9,
 * the default), kind 1 = the paper's ILU(0) in
 * red-black cell ordering (reading B12): x <- x + (L U)^{-1}(b - A x), undamped, nu steps
 * per stage, L U = the ILU(0) factors of the red-black permuted A.  The pivots are
 * recomputed from the operator's current transmissibilities at the start of every
 * msb_ms_iterate / msb_fgmres call.  Errors: MSB_EINVAL for another kind. */
msb_status msb_solver_set_smoother(msb_ctx ctx, msb_solver s, int32_t kind);

/* ---------------------------------------------------------------- FGMRES (§8 NEXT-1)
 * Flexible GMRES(restart) right-preconditioned by ONE multibasis cycle (Eq. 8 from x = 0)
 * over the solver's static levels followed, when one is installed (M_dyn > 0), by its
 * dynamic constant-basis stage — held fixed for the whole solve, as the paper builds
 * dynamic partitions from the most recent nonlinear iteration (reading
 * B6).  The paper's other outer solver.  Arnoldi with classical Gram-Schmidt applied twice,
 * Givens rotations on the host; stops when the Arnoldi residual estimate
 * |g_{j+1}| <= tol ||b|| (confirmed by the true residual at the restart boundary), at
 * max_iter (MSB_NOT_CONVERGED), or after exactly fixed_iters > 0 steps.
 * b, x: host|dev N doubles (NULL b = the operator's q; x in x0 / out x); restart in
 * [1, 64]; res_hist: host array of (max(max_iter, fixed_iters) + 2 + #restarts)
 * doubles or NULL (ρ_0, then the estimate after every step).  Workspace: (2 restart + 3) N
 * doubles of device memory for the call.  Errors: MSB_EINVAL (null handle, restart out of
 * range, no stage), MSB_ENOMEM, MSB_ECUDA; NaN in the Arnoldi estimate is not trapped
 * (the run ends at max_iter with MSB_NOT_CONVERGED). */
msb_status msb_fgmres(msb_ctx ctx, msb_solver s, const double* b, double* x, double tol,
                      int32_t restart, int32_t max_iter, int32_t fixed_iters, int32_t* iters_out,
                      double* res_hist);

/* ---------------------------------------------------------------- config-4 transport (row a12)
 * Face fluxes F_f = T_f (p_i - p_l) with T including the current mobility, and
 * explicit single-point-upstream transport of water saturation S (
 * readings A17, A18) over time dt in n_sub = ceil(dt / dt_cfl) equal sub-steps:
 *   S_i += h/(φ_i |Ω_i|) (Σ_in F f_w(S_up) - Σ_out F f_w(S_i) + q_i^+ - q_i^- f_w(S_i)),
 *   f_w = λ_w/λ_t, λ_w = S^2/μ_w, λ_o = (1-S)^2/μ_o,
 *   dt_cfl = 0.5 min_i φ_i|Ω_i| / (out_i * fw_max'),  out_i = Σ outflow + q_i^-.
 * Also writes the upstream total mobility per face (mob_out, compact face layout,
 * host|dev or NULL) for the next pressure step.  p, S, phi: dev arrays of N. */
msb_status msb_transport_upwind(msb_ctx ctx, msb_op op, const double* p, double* S,
                                const double* phi, double mu_w, double mu_o, double dt,
                                double* mob_out, int32_t* substeps_out);
/* Per-face upstream total mobility λ_t(S_up) = S^2/μ_w + (1-S)^2/μ_o, upstream by the
 * sign of p_i - p_l (ties to the left/lower cell; reading A17).
 * p, S: host|dev N doubles, or NULL for zero (step 1: S = 0 gives λ_t = 1/μ_o on every
 * face).  mob_out: host|dev, compact face layout.  Synchronises. */
msb_status msb_upstream_mobility(msb_ctx ctx, msb_op op, const double* p, const double* S,
                                 double mu_w, double mu_o, double* mob_out);
/* Config-4 pressure step length (reading A18): dt = pv_per_step * Σ_i φ_i |Ω_i| / Σ_i q_i^+
 * (0 without injection), summed on the device in a fixed order.  phi host|dev N doubles;
 * dt_out host.  Synchronises. */
msb_status msb_transport_step_size(msb_ctx ctx, msb_op op, const double* phi,
                                   double pv_per_step, double* dt_out);

/* ---------------------------------------------------------------- CPR two-stage (§8 NEXT-4)
 * Constrained-pressure-residual preconditioning of the fully implicit compressible
 * two-phase system (PAPER.md:122-203 §4, :287-292), readings C1-C6.
 * Model: phases w, o with one component each, no gravity / capillarity;
 * unknowns x = (p_1..p_N | S_1..S_N), S = S_w; equations F = (F_w | F_o),
 *   F_a^i = (φ ρ_a S_a)_i - (φ ρ_a S_a)_i^n + (Δt/|Ω_i|) Σ_faces T_f (ρ_a λ_a)_up (p_i - p_j)
 *           - (Δt/|Ω_i|) q_a^i,
 *   ρ_a(p) = rho_a exp(c_a (p - p_ref)), φ(p) = phi exp(c_r (p - p_ref)),
 *   λ_w = S^n/mu_w, λ_o = (1-S)^n/mu_o (n = nrel in {1, 2}), upstream cell = the face's
 *   left/lower cell when p_l >= p_r (reading A17); per-cell rate Q: Q > 0 injects water
 *   (q_w = ρ_w Q), Q < 0 produces at the cell's fractional flow (q_a = ρ_a f_a Q).
 * T_f = the operator's base transmissibility (K, cell sizes, multipliers; no mobility).
 * Jacobian storage (msb_cpr_export): 28 planes of N doubles, plane (2 b + v) * 7 + d holds
 * ∂F_b(c)/∂x_v(nb_d(c)) for b, v in {0 (w | p), 1 (o | S)} and stencil slot d = 0 centre,
 * 1 -x, 2 +x, 3 -y, 4 +y, 5 -z, 6 +z (0 where the neighbour does not exist). */
typedef struct msb_cpr_s* msb_cpr;
typedef struct {
  double mu_w, mu_o;    /* viscosities                                */
  double rho_w, rho_o;  /* densities at p_ref                         */
  double c_w, c_o, c_r; /* fluid and rock compressibilities           */
  double phi;           /* porosity at p_ref                          */
  double p_ref, dt;     /* reference pressure, time step Δt           */
  int32_t nrel;         /* relative-permeability exponent (1 or 2)    */
} msb_fluid;

/* Create a CPR object on `op` (grid + base T) whose predictor runs n_cycles Eq.-(8) cycles
 * (pre-smoothing damped Jacobi ω_s, ν = 1, then the coarse correction of `lev`) on
 * J*_pp ("one or a few cycles").  `lev` must be a Cartesian level of the same
 * grid (its smoothed basis P is used as prolongation, R = P^T; reading C5) with M <= 8192
 * (the predictor inverts A_c densely); it is not owned, must outlive the CPR object, and
 * must not be re-smoothed between msb_cpr_decouple and the applications that use it.
 * Errors: MSB_EINVAL (nrel, n_cycles < 1, explicit level, M > 8192, dt or a viscosity
 * <= 0), MSB_EDIM (other grid). */
msb_status msb_cpr_create(msb_ctx ctx, msb_op op, msb_level lev, const msb_fluid* fl,
                          int32_t n_cycles, double omega_s, msb_cpr* out);
/* Linearize at (p, S) with previous time level (p_n, S_n) (host|dev, N doubles each) and
 * per-cell well rates q (host|dev N doubles, or NULL = none): F and J on the device. */
msb_status msb_cpr_linearize(msb_ctx ctx, msb_cpr c, const double* p, const double* S,
                             const double* p_n, const double* S_n, const double* q);
/* Decouple: method 0 = no weights (w = (1, 0)), 1 = IMPES
 * (Σ_b W_b ∂A_b/∂S = 0), 2 = quasi-IMPES (Σ_b W_b diag ∂F_b/∂S = 0); per cell the system
 * [m_1 m_2; 1 1] w = [0; 1], w = (1, 0) where m_1 = m_2 = 0.  Then
 * J* = W J, F* = W F (first block row W_1 row_w + W_2 row_o, second row unchanged), the
 * predictor's coarse operator A_c = P^T J*_pp P (exact 128-bit fixed point) and its
 * explicit inverse (blocked Gauss–Jordan without pivoting on the fp64 tensor cores;
 * reading C5), and the corrector's ILU(0) of the full J* (2 x 2 cell blocks, red-black
 * cell order, reading C4).  Errors: MSB_ESINGULAR for a singular weight system, a coarse
 * pivot <= 1e-14 max|A_c| or a singular ILU(0) pivot block; MSB_EINVAL before linearize. */
msb_status msb_cpr_decouple(msb_ctx ctx, msb_cpr c, int32_t method);
/* dx = M_CPR^{-1} r: Δp = predictor(r_p); r' = r - J*[:, p] Δp;
 * dx = (Δp, 0) + (L U)^{-1} r'.  r, dx: dev, 2N doubles (may not alias). */
msb_status msb_cpr_apply(msb_ctx ctx, msb_cpr c, const double* r, double* dx);
/* y = J* x (dev, 2N doubles). */
msb_status msb_cpr_apply_system(msb_ctx ctx, msb_cpr c, const double* x, double* y);
/* Parity dumps (host|dev, NULL skips): F (2N), J (28 N planes, layout above), w (2N:
 * w_1 | w_2), F* (2N), J*'s first block row (14 N planes: pp slots 0..6 | ps slots 0..6). */
msb_status msb_cpr_export(msb_ctx ctx, msb_cpr c, double* F, double* J, double* w,
                          double* Fs, double* Js_row0);
/* The predictor's coarse operator A_c = P^T J*_pp P (dense M*M row-major, host|dev). */
msb_status msb_cpr_export_coarse(msb_ctx ctx, msb_cpr c, double* Ac, int32_t* M_out);
/* Flexible GMRES(restart) on J* dx = b (b host|dev 2N or NULL = -F*; x host|dev 2N, in x0,
 * out x), right-preconditioned by precond 1 = the CPR two-stage, 2 = the ILU(0) corrector
 * alone; same stopping rule and outputs as msb_fgmres. */
msb_status msb_cpr_fgmres(msb_ctx ctx, msb_cpr c, const double* b, double* x, double tol,
                          int32_t restart, int32_t max_iter, int32_t fixed_iters,
                          int32_t precond, int32_t* iters_out, double* res_hist);
msb_status msb_cpr_destroy(msb_cpr c);

#ifdef __cplusplus
}
#endif
#endif /* MSB_H */
