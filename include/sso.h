/*
 * sso.h — C ABI of the B200-native JAX-SSO hot path (arXiv 2407.20026).
 *
 * The path (BASELINE.json north_star):
 *   A0  pattern build      PAPER.md:82-83   (element_K_*_indices -> global positions)
 *   A1  element stiffness  PAPER.md:75-82, 112 (beam 12x12, MITC-4 quad 24x24)
 *   A2  assembly+supports  PAPER.md:58, 83-96 (vectorised scatter-add; Eq. 2-3 with b = 0)
 *   A3  Jacobi-PCG solve   PAPER.md:71-74 (Eq. 1 K u = f), BASELINE.json north_star
 *   A4  adjoint gradient   PAPER.md:212-221 (Eq. 5-6), objective PAPER.md:144, 252
 *
 * Conventions (DESIGN.md readings):
 *   - node ids are 0..n_nodes-1; element order is beams first, then quads;
 *   - DOF numbering node-major, component-minor: 6*node + c,
 *     c in (UX, UY, UZ, RX, RY, RZ);
 *   - supports: 6-bit mask per node, bit c set = DOF c fixed at 0 (b = 0);
 *     repeated nodes OR-merge; supports are applied by symmetric elimination;
 *   - every pointer passed to sso_create / sso_set_design is COPIED; the
 *     library owns all device state; outputs are written to caller-owned
 *     buffers of the stated sizes;
 *   - `mem` (sso_options.mem, changeable with sso_set_stream) says whether the
 *     f / u / gradient / design pointers of sso_set_design, sso_solve,
 *     sso_grad, sso_grad_at and sso_spmv are HOST or DEVICE pointers.  Device
 *     pointers must live on the handle's device.  All work is enqueued on the
 *     handle's CUDA stream; every call returns after that stream has completed
 *     its work unless stated otherwise;
 *   - one handle = one stream, not re-entrant; distinct handles are independent;
 *   - results are deterministic: same inputs -> bit-identical outputs
 *     (atomic-free, fixed-order reductions).
 *
 * Error behaviour: every int-returning call returns an sso_status; on failure
 * sso_last_error(h) (or sso_last_error(NULL) for sso_create) holds a message
 * naming the element / node / DOF at fault.  Device-side numeric failures
 * (degenerate element, singular diagonal, non-SPD, not converged) are
 * reported by the call that detects them.
 */
#ifndef SSO_H
#define SSO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sso_ctx* sso_handle;

typedef enum {
  SSO_OK = 0,
  SSO_E_INVALID = 1,        /* bad argument / input validation      */
  SSO_E_VALIDATION = 2,     /* reserved for CLI parity/FD threshold failures */
  SSO_E_NUMERIC = 3,        /* generic numeric failure                                     */
  SSO_E_DEGENERATE = 11,    /* zero-length beam, zero quad normal, det J <= 0 */
  SSO_E_SINGULAR = 31,      /* free DOF with diagonal <= 0                   */
  SSO_E_NOT_SPD = 32,       /* p^T K p <= 0 inside CG                                      */
  SSO_E_NOT_CONVERGED = 33, /* max_iter reached; u holds the last iterate, info filled     */
  SSO_E_CUDA = 40,
  SSO_E_NCCL = 41,
  SSO_E_OOM = 42,
  SSO_E_STATE = 43          /* call order violated (e.g. sso_grad before sso_solve)        */
} sso_status;

typedef enum {
  SSO_OBJ_COMPLIANCE = 0,     /* C = f^T u       (reading c2; s = 1)                       */
  SSO_OBJ_STRAIN_ENERGY = 1   /* g = 0.5 f^T u   (s = 1/2)              */
} sso_objective;

typedef enum { SSO_MEM_HOST = 0, SSO_MEM_DEVICE = 1 } sso_mem;

/* Mesh: SoA coordinates (fp64, n_nodes each); beam_conn [n_beams][2];
 * quad_conn [n_quads][4] in cyclic order.  Host pointers, copied. */
typedef struct {
  int32_t n_nodes;
  const double *x, *y, *z;
  int32_t n_beams;
  const int32_t* beam_conn;
  int32_t n_quads;
  const int32_t* quad_conn;
} sso_mesh;

/* Sections: A, Iy, Iz, J [n_beams] (may be NULL when n_beams == 0);
 * t [n_quads] shell thickness (may be NULL when n_quads == 0).  Host, copied. */
typedef struct {
  const double *A, *Iy, *Iz, *J;
  const double* t;
} sso_sections;

/* Materials per element (beams first, then quads): E, nu [n_beams + n_quads];
 * G may be NULL -> G = E / (2 (1 + nu)).  Host, copied. */
typedef struct {
  const double *E, *nu, *G;
} sso_materials;

/* Supports: n entries of (node, 6-bit mask), b = 0 (reading c1).  Host, copied. */
typedef struct {
  int32_t n;
  const int32_t* node;
  const uint8_t* mask6;
} sso_supports;

typedef struct {
  double rtol;            /* CG stop: |r|_2 <= rtol |f_bc|_2            (default 1e-10) */
  int64_t max_iter;       /* CG iteration cap                          (default 200000) */
  double drill_alpha;     /* drilling penalty gamma_d = alpha_d G      (default 1e-3)   */
  int32_t warm_start;     /* 1: sso_solve reads u as x0                (default 0)      */
  int32_t check_every;    /* CG iterations per device-side graph chunk (default 64)     */
  sso_mem mem;            /* pointer kind of solve/grad/design buffers (default HOST)   */
  void* cuda_stream;      /* cudaStream_t to enqueue on; NULL = library-owned stream    */
  int32_t device;         /* CUDA device ordinal                        (default: current) */
  /* Partitioning.  The node range is split into contiguous strips
   * part_ranges[0] = 0 < ... < part_ranges[P] = n_nodes (NULL = equal node counts).
   * nranks == 1, n_parts == P > 1: all P strips live in this handle on one GPU
   *   (in-process transport); buffers stay global.
   * nranks == P > 1: this handle is strip `rank` on its own GPU; halos and the CG
   *   scalars travel through NCCL (communicator from nccl_unique_id, 128 bytes, made
   *   by sso_nccl_unique_id on one rank and broadcast by the caller).  f, u and
   *   dC_dxyz then cover the rank's owned nodes only, dC_dt its owned quads (first
   *   node owned), in ascending global order; C is global.  (defaults: 1, NULL, 1, 0, NULL) */
  int32_t n_parts;
  const int32_t* part_ranges;
  int32_t nranks, rank;
  const void* nccl_unique_id;
  /* Batched designs: B >= 1 designs share connectivity,
   * supports and materials; each has its own coordinates, thicknesses, loads and CG
   * (own alpha / beta / convergence, run in lockstep in the same kernel launches).
   * With B > 1 (single strip, single rank only) every per-design buffer is
   * design-major: sso_set_design x, y, z [B][n_nodes], t [B][n_quads]; sso_solve f, u
   * [B][6 n_nodes], info [B]; sso_grad C [B], dC_dxyz [B][3][n_nodes], dC_dt
   * [B][n_quads]; sso_grad_at / sso_spmv [B][6 n_nodes].  Exports show design 0. */
  int32_t batch;
  /* Residual reliability (reading c10): 0 = plain recurrence; 1 (default) = when the
   * recurrence residual meets rtol, recompute f - K u and restart CG (p = z, at most
   * twice) if the true residual exceeds 2 rtol, unless it sits at the fp64 floor of
   * K u; 2 = also replace r by f - K u each time |r|^2 fell 1e4x (reliable updates). */
  int32_t reliable;
  /* 0 (default) = element stiffness and assembly fused in one pass (no staged element
   * matrices) when the mesh is quad-only with node degree <= 10; 1 = always the staged
   * path (element kernel, then the segmented-sum gather). */
  int32_t assembly;
  /* 0 (default) = storage 3.  1 = full CSR storage (row-major runs of 36 deg values per node).
   * 3 = upper node blocks (n, m >= n) of the symmetric K_bc only (44 % fewer value bytes on
   * shell grids), each one contiguous 38-double record (36 values as nine 2x2 sub-blocks + 2
   * zero pads), and a ONE-pass "pull" SpMV: the CTA that owns a chunk of row nodes streams
   * their upper runs (one bulk copy) and the stored blocks (n, m) of their lower neighbours
   * n < m (one TMA gather4 per node; an L2 hit: chunks are dealt round-robin, so the owner
   * streams them in the same window) and forms
   * y_m = sum_{j>=m} K_mj x_j + sum_{n<m} K_nm^T x_n.  Storage 3 also applies to strips
   * (owned nodes precede halo nodes locally, so lower neighbours are owned).  Exports return
   * the full CSR.  Other values (including the retired 2) -> SSO_E_INVALID. */
  int32_t storage;
  /* Preconditioner of the CG (reading c10 / c19): 0 (default) = point Jacobi, M =
   * diag(K_bc) (the north star's); 1 = node-block Jacobi, M = blockdiag(K_nn) of the 6x6
   * diagonal block of every node (inverted once per sso_assemble; about 30 % fewer
   * iterations on shells). */
  int32_t precond;
} sso_options;

typedef struct {
  int64_t iters;          /* CG iterations performed                                   */
  double rel_res;         /* recurrence residual |r|/|f_bc| at exit                    */
  double true_rel_res;    /* |f_bc - K_bc u| / |f_bc| recomputed at exit               */
  double ms;              /* device time of the solve (CUDA events)                    */
  int32_t status;         /* sso_status of this solve                                  */
  /* Certification (Eq. 1 solved by CG).  CG from
   * x0 = 0 is the Lanczos process on M^-1 K: its coefficients form the tridiagonal
   * T[k][k] = 1/alpha_k + beta_{k-1}/alpha_{k-1}, T[k][k+1] = sqrt(beta_k)/alpha_k, whose
   * extreme eigenvalues (Ritz values; formed on the device by Sturm multisection) lie
   * inside the spectrum of M^-1 K.  lanczos_iters = coefficients used (the first CG
   * segment, at most 2^18; a restart starts a new sequence).  With r = f_bc - K u the
   * TRUE residual, rz = r^T M^-1 r, C = f_bc^T u = |u|_K^2 and m_min <= lambda_min(M)
   * (min 1/dinv, or min over nodes of 1/|(K_nn)^-1|_F for precond 1):
   *   err_energy_est = sqrt(rz / (lanczos_lmin C))                    >= |e|_K / |u|_K
   *   err2_est       = sqrt(rz) / (lanczos_lmin sqrt(m_min)) / |u|_2   >= |e|_2 / |u|_2
   * where ">=" holds with the exact lambda_min(M^-1 K) in place of lanczos_lmin (which is
   * an upper estimate of it: the figures are estimates, exact once CG has resolved the
   * smallest eigenvalue).  NaN when undefined (no iterations, C <= 0). */
  int32_t lanczos_iters;
  double lanczos_lmin, lanczos_lmax;
  double err_energy_est, err2_est;
} sso_solve_info;

/* Fill *o with the defaults listed above.  Always SSO_OK. */
int sso_options_default(sso_options* o);

/* Validate, build the node-block CSR pattern (A0), upload all inputs.
 * Errors: SSO_E_INVALID (index out of range, i_node == j_node, E/G/A/Iy/Iz/J/t <= 0,
 * nu outside [0, 0.5), repeated node in a quad, non-finite input, no supports or an
 * all-zero mask), SSO_E_DEGENERATE (zero-length beam), SSO_E_CUDA / SSO_E_OOM.
 * On error *out is NULL and sso_last_error(NULL) explains. */
int sso_create(const sso_mesh* mesh, const sso_sections* sec, const sso_materials* mat,
               const sso_supports* sup, const sso_options* opt, sso_handle* out);

/* Replace design variables: x, y, z [n_nodes] and/or t [n_quads]; NULL = unchanged.
 * Pointer kind per `mem`.  Invalidates the assembled K (call sso_assemble again). */
int sso_set_design(sso_handle h, const double* x, const double* y, const double* z,
                   const double* t);

/* Change the stream and pointer kind used by subsequent calls. */
int sso_set_stream(sso_handle h, void* cuda_stream, sso_mem mem);

/* A1 + A2: element stiffness for all elements, segmented-sum assembly into the fixed
 * CSR values (layout per sso_options.storage), supports by elimination, Jacobi diagonal
 * (and, with precond = 1, the inverse 6x6 node blocks).  Errors: SSO_E_DEGENERATE
 * (element id in the message), SSO_E_SINGULAR (free DOF with diagonal <= 0 or a node
 * block that is not positive definite). */
int sso_assemble(sso_handle h);

/* A3: Jacobi-PCG (point or node-block, sso_options.precond) on K_bc u = f_bc to
 * |r| <= rtol |f_bc|.  f [6 n_nodes] (entries at constrained DOFs ignored),
 * u [6 n_nodes] output (zeros at constrained DOFs); read as x0 when warm_start.
 * info may be NULL ([batch] entries otherwise).  Errors: SSO_E_STATE (not assembled),
 * SSO_E_NOT_SPD, SSO_E_NOT_CONVERGED (u = last iterate). */
int sso_solve(sso_handle h, const double* f, double* u, sso_solve_info* info);

/* A4: objective and adjoint gradient at the last solve's (f, u):
 * C [1]; dC_dxyz [3][n_nodes] (SoA: all x, then y, then z); dC_dt [n_quads].
 * Any output pointer may be NULL to skip it.  Errors: SSO_E_STATE (no solve yet). */
int sso_grad(sso_handle h, sso_objective obj, double* C, double* dC_dxyz, double* dC_dt);

/* A4 at a caller-given state: C = s f^T u and -s sum_e u_e^T dK_e/dp u_e for the given
 * f, u [6 n_nodes] (u taken as is, including constrained entries).  Pointer kind per mem. */
int sso_grad_at(sso_handle h, sso_objective obj, const double* f, const double* u,
                double* C, double* dC_dxyz, double* dC_dt);

/* General objective g(u, p) (Eq. 5-6):
 * sso_adjoint_solve solves K_bc^T lambda = dg/du (K symmetric; entries at constrained
 * DOFs ignored, lambda = 0 there) with the same Jacobi-PCG and options as sso_solve,
 * keeping the primal state (u, f) of the last solve.  dg_du, lambda [6 n_nodes].
 * sso_grad_adjoint then returns the Eq. 6 term -lambda^T (dK/dp) u at the primal u
 * (df/dp = 0, reading c3) for p = coordinates dg_dxyz [3][n_nodes], thicknesses
 * dg_dt [n_quads] and moduli dg_dE [n_beams + n_quads] (any may be NULL); the caller
 * adds the explicit dg/dp.  Single-strip handles; a batch solves every design's adjoint in
 * the same batched PCG (dg_du, lambda [batch][6 n_nodes], info [batch]; gradients with a
 * leading design axis).  The term is formed in one pass of the gradient kernels in bilinear
 * form (strains of lambda and u, dual numbers through lambda_e^T K_e(p) u_e). */
int sso_adjoint_solve(sso_handle h, const double* dg_du, double* lambda, sso_solve_info* info);
int sso_grad_adjoint(sso_handle h, const double* lambda, double* dg_dxyz, double* dg_dt, double* dg_dE);

/* SIMP / material design variable (Eq. 12):
 * dC_dE [batch][n_beams + n_quads] = -s u_e^T (dK_e/dE_e) u_e at the last solve, where the
 * element's whole elastic tensor scales with E_e (a given G scales with it).  With
 * E_e = rho_e^P E0_e the caller forms dC/drho = dC/dE * P rho^(P-1) E0.  Single-strip
 * handles.  Errors: SSO_E_STATE (no solve yet). */
int sso_grad_E(sso_handle h, sso_objective obj, double* dC_dE);

/* SIMP density design variable (Eq. 12:
 * E_j = p_T,j^P E_*,j).  rho, E0 [n_beams + n_quads] (beams first, shared by a batch;
 * pointer kind per mem): the element moduli become E_e = rho_e^P E0_e on the device, and
 * G_e = rho_e^P G0_e when G0 [n_beams + n_quads] is given, else E_e / (2 (1 + nu_e)).
 * sso_grad_density then returns dC_drho [batch][n_beams + n_quads] =
 * dC/dE_e * P rho_e^(P-1) E0_e at the last solve (the chain rule of Eq. 12 applied on the
 * device to sso_grad_E's dC/dE).  Invalidates the assembly; sso_set_material ends the
 * density mode.  Single-strip handles.  Errors: SSO_E_INVALID (rho outside (0, 1],
 * P < 1, E0 / G0 <= 0 or non-finite), SSO_E_STATE (grad without a density or a solve). */
int sso_set_density(sso_handle h, const double* rho, double penal, const double* E0, const double* G0);
int sso_grad_density(sso_handle h, sso_objective obj, double* dC_drho);

/* Replace the element moduli E [n_beams + n_quads] (shared by a batch; pointer kind per
 * mem); G follows (derived G recomputed, given G scaled).  Invalidates the assembly.
 * Single-strip handles.  Errors: SSO_E_INVALID (E <= 0). */
int sso_set_material(sso_handle h, const double* E);

/* Prescribed support displacements (Eqs. 2-3
 * V u = b with b != 0; reading c18 in DESIGN.md).  b: [6 n_nodes] fp64, pointer kind per
 * mem; only the entries of constrained DOFs are used (the rest ignored); NULL switches
 * them off.  Solved by lifting: K_ff u_f = f_f - K_fc b, u_c = b (K_fc b from one extra
 * unconstrained assembly + SpMV inside the next sso_assemble, which this call requires).
 * While active, sso_grad / sso_grad_E return the compliance gradient C = s f^T u,
 * dC/dp = -lambda^T dK/dp u + (lambda + s u)^T df/dp with lambda = s u_hom (the same loads
 * with b = 0: one more PCG solve inside sso_grad); sso_grad_at is refused.
 * Single-strip handles; a batch takes one b per design ([batch][6 n_nodes]; not combined
 * with area loads).  Errors: SSO_E_INVALID (non-finite b, partitioned handle). */
int sso_set_prescribed(sso_handle h, const double* b);

/* Design-dependent area loads (Eq. 6 with
 * df/dp != 0; reading c17 in DESIGN.md).  Every quad e carries the load per unit area
 * (q[e] + w[e] t_e) in the direction dir[3], lumped equally to its 4 nodes with
 * A_e = 1/2 |(X3 - X1) x (X4 - X2)| at the CURRENT design:
 *     f_n[0:3] += dir (q[e] + w[e] t_e) A_e / 4.
 * q: pressure-like load per unit area, w: unit weight (rho g; w t is self-weight); both
 * [n_quads] global, pointer kind per mem (either may be NULL = zeros; both NULL switches
 * the area load off); dir: HOST pointer, 3 doubles, not normalised.  While active:
 *   - sso_solve adds the area load to f (f may then be NULL = no nodal loads);
 *   - sso_grad / sso_grad_at return dC/dp = s (2 u^T df/dp - u^T dK/dp u) (sso_grad_at
 *     expects the f it is given to include the area load);
 *   - sso_grad_adjoint returns -lambda^T (dK/dp u - df/dp);
 *   - sso_adjoint_solve solves with dg/du alone.
 * Beams carry no area load.  Errors: SSO_E_INVALID (non-finite values, dir NULL). */
int sso_set_area_load(sso_handle h, const double* q, const double* w, const double* dir);

/* Hat filter of sensitivities ("a standard hat filter with a
 * radius of r"; reading c16 in DESIGN.md):
 *     out_i = sum_j w_ij in_j / sum_j w_ij,   w_ij = max(0, radius - |X_i - X_j|),
 * X = the current node coordinates (on_elements = 0; n = n_nodes) or the element
 * centroids, beams then quads, each the mean of its nodes (on_elements != 0;
 * n = n_beams + n_quads).  in, out: [ncomp][n] fp64, ncomp in 1..3 (e.g. the three rows of
 * dC/dxyz), pointer kind per mem; out may not alias in.  The neighbour cell grid is
 * cached per (kind, radius) and rebuilt after sso_set_design changes coordinates.  A batch
 * filters every design over its own coordinates (in, out [batch][ncomp][n]; the designs'
 * grids are built per call).  Single-strip handles.  Errors: SSO_E_INVALID (radius <= 0 or
 * non-finite, ncomp out of range, NULL pointers, partitioned handle). */
int sso_hat_filter(sso_handle h, int32_t on_elements, double radius, int32_t ncomp, const double* in,
                   double* out);

/* y = K_bc x with the assembled matrix (x, y [6 n_nodes]; pointer kind per mem). */
int sso_spmv(sso_handle h, const double* x, double* y);

/* Sizes: ndof = 6 n_nodes; nnz of the scalar CSR; node blocks of the node graph. */
int sso_sizes(sso_handle h, int64_t* ndof, int64_t* nnz, int64_t* n_blocks);

/* Debug / parity exports (HOST pointers always; caller-allocated):
 *   row_ptr [ndof+1] int64, col_idx [nnz] int32, vals [nnz] fp64 (any may be NULL);
 *   block_rank: beams [n_beams][4] then quads [n_quads][16], int32: position of
 *     element node j in the sorted node adjacency of element node i (i-major);
 *   ke: staged element matrices of elements [first, first+count) in the global
 *     element order, each dense row-major in element DOF order (144 or 576 fp64);
 *   dinv [ndof]: Jacobi inverse diagonal of K_bc. */
int sso_export_csr(sso_handle h, int64_t* row_ptr, int32_t* col_idx, double* vals);
int sso_export_scatter(sso_handle h, int32_t* block_rank);
int sso_export_ke(sso_handle h, int64_t first, int64_t count, double* ke);
int sso_export_dinv(sso_handle h, double* dinv);

/* Device storage of the assembled matrix: stored values / node blocks (owned rows) and
 * the layout in use: *symmetric = 0 full storage, 3 upper blocks (38-double records of 2x2
 * sub-blocks) with the one-pass pull SpMV.  stored_values counts the 36 values per block (not the record pads). */
int sso_storage_info(sso_handle h, int64_t* stored_values, int64_t* stored_blocks, int32_t* symmetric);


/* Partition of this handle: number of strips held, first owned global node, owned
 * node count and owned quad count (the extents of the caller's f / u / gradients). */
int sso_part_info(sso_handle h, int32_t* n_parts_here, int32_t* own_node_begin, int32_t* own_nodes,
                  int32_t* own_quads);

/* ncclGetUniqueId through the library's run-time NCCL binding (out: 128 bytes). */
int sso_nccl_unique_id(void* out);

/* Host-only partition queries (no GPU needed; the multi-process CPU tests use them).
 * Rank-local CSR pattern of strip `part` (rows of its owned nodes, global column ids):
 * call with row_ptr = col_idx = NULL to get *nnz, then with [6 n_own + 1] / [nnz] buffers.
 * The strips' patterns concatenate to the global pattern. */
int sso_local_pattern(const sso_mesh* mesh, const int32_t* ranges, int32_t n_parts, int32_t part,
                      int64_t* nnz, int64_t* row_ptr, int32_t* col_idx);
/* Halo plan of strip `part`: halo node ids (global, ordered by owner then id), the
 * neighbour strips and, per neighbour, the owned nodes sent to it (in its halo order).
 * Call with NULL arrays to get *n_halo and *n_nbrs; send_gid holds sum(send_count). */
int sso_halo_plan(const sso_mesh* mesh, const int32_t* ranges, int32_t n_parts, int32_t part,
                  int32_t* n_halo, int32_t* halo_gid, int32_t* n_nbrs, int32_t* nbr_part,
                  int32_t* send_count, int32_t* send_gid);

/* Kernel timing with CUDA events recorded on the handle's stream while enabled.
 * names: "element", "assemble", "spmv", "update", "grad", "reduce".  Outside the
 * CG loop every launch of the family is bracketed; inside sso_solve's CG loop
 * (graph replays) every 16th SpMV launch is bracketed by event nodes (a live
 * sample; the cost stays below 0.5 % of the solve).  total_ms and launches cover
 * the timed launches and accumulate since the last reset. */
int sso_profile_enable(sso_handle h, int32_t on);
int sso_profile_read(sso_handle h, const char* name, double* total_ms, int64_t* launches);
int sso_profile_reset(sso_handle h);

/* Number of kernel launches issued by the library since the handle was created
 * (graph-launched kernels counted individually). */
int64_t sso_launch_count(sso_handle h);

const char* sso_last_error(sso_handle h);
void sso_destroy(sso_handle h);

#ifdef __cplusplus
}
#endif
#endif /* SSO_H */
