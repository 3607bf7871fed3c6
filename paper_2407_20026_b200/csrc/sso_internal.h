// Internal declarations of the B200 JAX-SSO hot-path library (not part of the ABI).
#pragma once
#include <cstdlib>
#include <utility>

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "sso.h"

namespace sso {

// ---------------------------------------------------------------------------
// Host-side pattern (A0).  Node-block CSR: node n has deg(n) = node_ptr[n+1] -
// node_ptr[n] neighbours node_col[node_ptr[n] ..] (ascending, incl. n).  The
// scalar CSR is implied: row 6n+a holds columns 6m+b for m in adj(n), b = 0..5,
// row_ptr[6n+a] = 36 node_ptr[n] + 6 a deg(n); the values of node n's six rows
// are contiguous at 36 node_ptr[n].
// ---------------------------------------------------------------------------
struct HostPattern {
  int32_t n_nodes = 0, n_beams = 0, n_quads = 0;
  std::vector<int64_t> node_ptr;      // [n_nodes+1]
  std::vector<int32_t> node_col;      // [n_blocks]
  std::vector<int32_t> block_rank;    // beams [Eb][4], quads [Eq][16]
  std::vector<int64_t> contrib_ptr;   // [n_blocks+1]
  std::vector<int32_t> contrib;       // staged block ids, ascending (e, i, j)
  std::vector<int64_t> inc_ptr;       // [n_nodes+1] node -> element-node slots
  std::vector<int32_t> inc_slot;      // slot = 2e+i (beams) or 2Eb+4q+i (quads), ascending e
  int64_t n_blocks() const { return (int64_t)node_col.size(); }
  int64_t nnz() const { return 36 * n_blocks(); }
  int64_t n_staged_blocks() const { return 4 * (int64_t)n_beams + 16 * (int64_t)n_quads; }
};

// Upper-triangular (symmetric) node-block storage: node n keeps only the blocks
// (n, m) with m >= n (the diagonal block first).  Node m's incoming blocks (n, m),
// n < m, are lpull[lptr[m] ..] in ascending source node n (the pull SpMV).
struct UpperPattern {
  std::vector<int64_t> uptr;          // [n_nodes+1]
  std::vector<int32_t> ucol;          // [n_ublocks]
  std::vector<int32_t> urank;         // beams [Eb][4], quads [Eq][16]: rank in ucol(node_i) or -1
  std::vector<int64_t> ucontrib_ptr;  // [n_ublocks+1]
  std::vector<int32_t> ucontrib;      // staged block ids of upper blocks, ascending (e, i, j)
  std::vector<int64_t> lptr;          // [n_nodes+1] incoming blocks per node
  std::vector<int32_t> lpull;         // [2 * incoming]: (source node n, upper block index of (n, m))
  int64_t n_ublocks() const { return (int64_t)ucol.size(); }
};
void build_upper(const HostPattern& P, const int32_t* beam_conn, const int32_t* quad_conn,
                 UpperPattern& U);

// Builds the pattern; returns empty string on success, else an error message.
std::string build_pattern(int32_t n_nodes, int32_t n_beams, const int32_t* beam_conn,
                          int32_t n_quads, const int32_t* quad_conn, HostPattern& P);

// ---------------------------------------------------------------------------
// Device state shared by the PCG kernels (one instance in device memory).
// ---------------------------------------------------------------------------
struct CgState {
  double rz;        // r^T z (current)
  double pq;        // p^T K p (current iteration)
  double alpha, beta;
  double rr;        // r^T r
  double ff;        // f^T f
  double tol2;      // (rtol^2) * ff
  long long iter;
  long long max_iter;
  int done;         // 1 = converged or failed: all later kernels return immediately
  int status;       // sso_status
  unsigned int ticket[4];  // last-block-done counters (one per reduction site)
  int dist;         // 1 = partitioned: the SpMV writes its local p^T q piece to red[0] (the
                    //     single-reduction CG of cg_sr.cu allreduces red[] across parts)
  int act;         // residual replacement selected for this design (see cg_check)
  double red[4];    // local (then global) reduction values
  double rr_ref;    // r^T r at the last residual replacement
  double rz_prev;   // r^T z of the previous iteration (beta after a replacement)
  int restarts;     // final true-residual restarts used
  int floor;        // 1 = the true residual sits far above the recurrence (fp64 floor):
                    //     no further replacements / restarts
  int pfix;         // 1 = r was replaced after the fused update formed p: re-form p
  unsigned int arrive;  // fused update: CTAs arrived (monotonic, +grid per launch)
  int defer_alpha;  // 1 = the SpMV leaves its p^T q partials (partial + PQ_OFF) and the fused
                    //     update forms p^T q and alpha in every CTA (no last-CTA tail)
  int npq;          // number of those partials (the SpMV grid)
  // Lanczos history of the CG coefficients (Eq. 1 solved by CG; SURVEY
  // §8(c) C5 "extract Lanczos extreme Ritz values from (alpha, beta)"): (alpha_k, beta_k) of
  // every iteration of the first CG segment (recording stops at a restart), [lz_cap][2];
  // lanczos.cu forms the extreme Ritz values of M^-1 K from it.
  double* lz;
  int lz_cap, lz_n, lz_frozen;
  double lz_min, lz_max;
  // single-reduction CG of partitioned handles (cg_sr.cu): rtol^2 (tol2 becomes rtol^2 |f_bc|^2
  // once |f_bc|^2 is known, ff < 0 until then) and a restart flag (beta = 0 next)
  double tol2_rel;
  int sr_restart;
};

#ifdef __CUDACC__
// Record iteration k's (alpha_k, beta_k); called by the one thread that completes an
// iteration (fused update CTA 0, the last CTA of the classic update, cg_scalar_kernel).
__device__ __forceinline__ void lz_record(CgState* st, double alpha, double beta) {
  if (st->lz && !st->lz_frozen && st->lz_n < st->lz_cap) {
    st->lz[2 * st->lz_n] = alpha;
    st->lz[2 * st->lz_n + 1] = beta;
    st->lz_n += 1;
  }
}
#endif

// error flags written by device kernels (atomicMin on the offending index)
struct DevFlags {
  int degenerate_elem;   // INT_MAX = none
  int singular_dof;      // INT_MAX = none
};

// Kernel-family timers
enum Family { F_ELEMENT = 0, F_ASSEMBLE, F_SPMV, F_UPDATE, F_GRAD, F_REDUCE, F_COUNT };

struct Timers {
  bool on = false;
  double total_ms[F_COUNT] = {0};
  long long launches[F_COUNT] = {0};
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
};

// Batched designs: B designs share connectivity, supports and
// materials; per-design arrays are design-major with these strides (elements of
// the array type).  Kernels take the design from blockIdx.y.  B = 1: strides unused.
struct BatchStrides {
  int B = 1;
  int64_t node = 0;     // coordinates [B][n]
  int64_t quad = 0;     // thickness, dC/dt [B][n_quads]
  int64_t stage = 0;    // staged element blocks [B][36 n_staged]
  int64_t nnz = 0;      // CSR values [B][nnz]
  int64_t dof = 0;      // vectors [B][6 n]
  int64_t partial = 0;  // per-CTA partials [B][..]
  int64_t slot = 0;     // gradient slot partials [B][3 n_slots]
};

// Launch wrappers (implemented in the .cu files).  All are stream-ordered.
void launch_beam_elements(cudaStream_t s, int n_beams, const double* x, const double* y,
                          const double* z, const int32_t* conn, const double* A,
                          const double* Iy, const double* Iz, const double* J,
                          const double* E, const double* G, double* stage, DevFlags* flags,
    const BatchStrides& bs = BatchStrides());
void launch_quad_elements(cudaStream_t s, int n_quads, const double* x, const double* y,
                          const double* z, const int32_t* conn, const double* t,
                          const double* E, const double* nu, double drill_alpha,
                          double* stage, DevFlags* flags,
    const BatchStrides& bs = BatchStrides());
void launch_assemble(cudaStream_t s, int n_nodes, const int64_t* node_ptr,
                     const int32_t* node_col, const int64_t* contrib_ptr,
                     const int32_t* contrib, const double* stage, const uint8_t* fixed_mask,
                     double* vals, double* dinv, DevFlags* flags,
    const BatchStrides& bs = BatchStrides(), int cm = 0);

// Fused element stiffness + assembly for quad-only meshes (no staging).
int fused_max_degree();
void launch_quad_assemble_fused(cudaStream_t s, int n_own, int inc_pad, const int64_t* node_ptr,
                                const int32_t* node_col, const int32_t* inc_rec, const double* x,
                                const double* y, const double* z, const double* t, const double* E,
                                const double* nu, double drill_alpha, const uint8_t* fixed_mask,
                                double* vals, double* dinv, DevFlags* flags,
                                const BatchStrides& bs = BatchStrides(), int cm = 0);

// PCG kernels
int cg_grid();  // persistent grid size (multiple of the SM count)
void launch_cg_init(cudaStream_t s, int ndof, const double* f, const uint8_t* fixed_mask,
                    const double* dinv, double* fbc, double* x, double* r, double* p,
                    double* partial, CgState* st, int warm, const double* Kx0,
    const BatchStrides& bs = BatchStrides());
void launch_spmv_dot(cudaStream_t s, int n_nodes, const int64_t* node_ptr,
                     const int32_t* node_col, const double* vals, const double* p,
                     double* q, double* partial, CgState* st,
    const BatchStrides& bs = BatchStrides());
void launch_cg_update(cudaStream_t s, int ndof, const double* dinv, double* x, double* r,
                      const double* p, const double* q, double* partial, CgState* st,
    const BatchStrides& bs = BatchStrides());
void launch_cg_pupdate(cudaStream_t s, int ndof, const double* dinv, const double* r,
                       double* p, CgState* st,
    const BatchStrides& bs = BatchStrides());
// Fused x / r update + p update (one part, point Jacobi, B <= cg_fused_grid()): one
// kernel with a grid-wide barrier between the r^T z reduction and p_next = z + beta p
// (ping-pong p buffers, so a residual replacement can re-form p from the previous one).
void launch_cg_update_fused(cudaStream_t s, int ndof, const double* dinv, double* x, double* r,
                            const double* p, const double* q, double* pn, double* partial, CgState* st,
                            const BatchStrides& bs);
// p_out = dinv r + beta p_in after a residual replacement (st->pfix), else nothing.
void launch_cg_pfix(cudaStream_t s, int ndof, const double* dinv, const double* r, const double* pin,
                    double* pout, const CgState* st, const BatchStrides& bs);
// largest co-resident grid of the fused update kernel (0 = unavailable)
int cg_fused_grid();
// node-block Jacobi forms (block_jacobi.cu): the fused update and the p re-form
// from z after a residual replacement
void launch_cg_update_block_fused(cudaStream_t s, int n_nodes, const double* binv, double* x, double* r,
                                  const double* p, const double* q, double* pn, double* partial, CgState* st,
                                  const BatchStrides& bs);
void launch_cg_pfix_z(cudaStream_t s, int ndof, const double* z, const double* pin, double* pout,
                      const CgState* st, const BatchStrides& bs);
int cg_block_fused_grid();
// Cluster-resident PCG for small models (cg_small.cu): `iters` iterations of the
// single-reduction point-Jacobi recurrence, one thread-block cluster (<= 16 CTAs) per design,
// over the storage-3 records; s_vec (the fused path's second p buffer) keeps s = K p between
// chunks.
// cg_small_fits: the model fits one cluster (<= 1 152 nodes; the caller also requires every
// node to fit the pull descriptor: <= 5 upper and <= 4 pulled blocks).
bool cg_small_fits(int n_nodes);
void launch_cg_small(cudaStream_t s, int n_nodes, int iters, const int32_t* pdesc, const double* vals,
                     const double* dinv, double* x, double* r, double* p, double* s_vec, CgState* st,
                     const BatchStrides& bs);
// true the first time it is called for the current device with this mask (kernel attributes
// are per device: a process may hold handles on several GPUs)
inline bool first_on_device(uint64_t& mask) {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) d = 0;
  const uint64_t bit = 1ull << d;
  if (mask & bit) return false;
  mask |= bit;
  return true;
}
// Symmetric pull SpMV (storage 3): upper node blocks stored column-major per run;
// the row-owner warp streams its upper run and the upper blocks (n, m) of its lower
// neighbours (pull list lpull = [(n, upper block index)] per node, via lptr) and
// forms y = K x in one pass.  With st != nullptr also p^T q and alpha (CG).
// In-process parts in ONE launch (grid.y = part): each part's SpMV operands, its own tensor map
// (global memory, 64-byte aligned) and owned row count.
struct alignas(64) PullPart {
  CUtensorMap tmap;
  const int32_t* pdesc;
  const int32_t* ucol;
  const int2* lpull;
  const double* vals;
  const double* x;
  double* y;
  double* partial;
  CgState* st;
  int n_nodes;
  int pad_[3];
};
// y = K x with p^T q pieces into st->red[0] for every part of `mp` (device array of n_parts).
void launch_spmv_pull_multi(cudaStream_t s, const PullPart* mp, int n_parts, int max_nodes);
// Rows [node0, n_nodes) (default: all owned rows); on partitioned handles (st->dist) the
// p^T q piece is written to st->red[0] (red_add = 0) or added to it (red_add = 1).  share > 1:
// the launch runs concurrently with share - 1 others (in-process parts on their own streams)
// and takes 1/share of the persistent grid, so the parts run side by side on disjoint SMs.
void launch_spmv_pull(cudaStream_t s, const CUtensorMap* tmap, int n_nodes, int rows_per_design,
                      const int32_t* pdesc, const int32_t* ucol, const int32_t* lpull, const double* vals,
                      const double* x, double* y, double* partial, CgState* st,
                      const BatchStrides& bs = BatchStrides(), int node0 = 0, int red_add = 0, int share = 1);
// Storage 3 stores each upper 6x6 block as a record of PULL_BLOCK doubles: the nine 2x2
// sub-blocks (A, B) = K[2A..2A+1][2B..2B+1], 4 doubles each (column-major inside), sub-block
// 3B + A in slot PULL_SUB_POS nibble, and one 16-byte zero pad word (an odd 19-word record
// stride, see pcg.cu) placed before slot PULL_SUB_GAP.  A 16-byte half of a sub-block is a (row pair, one column) of K -- a row-pair
// product for the block's own row node and, with its neighbour half, a column-pair product of
// K^T for its column node: the same loads and FMA chains serve both (branch-free consumers).
constexpr int PULL_BLOCK = 38;
// offset of the SpMV's p^T q partials inside a design's partial buffer (16 cg_grid() doubles)
// when the fused update forms alpha (CgState::defer_alpha); SpMV grids stay below it
constexpr int PQ_OFF = 4096;
// sub-block 3B + A -> slot (nibble), and the pad word sits before slot PULL_SUB_GAP: the
// pair searched with tools/pull_perm_anneal.c together with the consumer lane table
constexpr unsigned long long PULL_SUB_POS = 0x830741652ull;
constexpr int PULL_SUB_GAP = 3;
// double offset of sub-block s inside a record
__host__ __device__ constexpr int pull_sub_off(int s) {
  return 4 * (int)((PULL_SUB_POS >> (4 * s)) & 15) + (((int)((PULL_SUB_POS >> (4 * s)) & 15) >= PULL_SUB_GAP) ? 2 : 0);
}
// offset of K[a][b] inside a record
__host__ __device__ constexpr int rec_off(int a, int b) {
  return pull_sub_off(3 * (b >> 1) + (a >> 1)) + 2 * (b & 1) + (a & 1);
}
// 16-int per-node descriptors of the pull SpMV (see pcg.cu)
void build_pull_desc(const UpperPattern& U, std::vector<int32_t>& desc);
// TMA map of the [rows][36] fp64 view of the values (gather4 of pulled blocks); 0 on success
int make_pull_tmap(const double* vals, int64_t rows, CUtensorMap* out);
void launch_spmv(cudaStream_t s, int n_nodes, const int64_t* node_ptr,
                 const int32_t* node_col, const double* vals, const double* x, double* y,
    const BatchStrides& bs = BatchStrides());
// Node-block Jacobi preconditioner (sso_options.precond = 1, block_jacobi.cu).  binv
// [B][21][n] packed upper triangles of (K_nn)^-1; layout 0 full runs, 3 upper-block records.
void launch_block_inverse(cudaStream_t s, int n_nodes, const int64_t* node_ptr, const int32_t* node_col,
                          const double* vals, int layout, double* binv, DevFlags* flags,
                          const BatchStrides& bs = BatchStrides());
void launch_cg_init_block(cudaStream_t s, int n_nodes, const double* f, const uint8_t* fixed_mask,
                          const double* binv, double* fbc, double* x, double* r, double* p, double* z,
                          double* partial, CgState* st, int warm, const double* Kx0,
                          const BatchStrides& bs = BatchStrides());
void launch_cg_update_block(cudaStream_t s, int n_nodes, const double* binv, double* x, double* r,
                            const double* p, const double* q, double* z, double* partial, CgState* st,
                            const BatchStrides& bs = BatchStrides());
void launch_cg_pupdate_z(cudaStream_t s, int ndof, const double* z, double* p, CgState* st,
                         const BatchStrides& bs = BatchStrides());
void launch_cg_replace_block(cudaStream_t s, int n_nodes, const double* fbc, const double* Kx, const double* binv,
                             double* r, double* z, double* partial, CgState* st, int mode,
                             const BatchStrides& bs = BatchStrides());
// Single-reduction Jacobi-PCG of partitioned handles (cg_sr.cu; Chronopoulos & Gear):
// per iteration halo(u) -> w = K u (SpMV, delta = u^T w into red[0]) -> ONE allreduce of
// red[0..3] -> update (alpha, beta from gamma = r^T u, delta; p = u + beta p, s = w + beta s,
// x += alpha p, r -= alpha s, u = M^-1 r; local gamma, r^T r into red[1], red[2]).  binv !=
// nullptr: node-block M.  init: f_bc, r = f_bc - K x0, u = M^-1 r, p = s = 0, red[1..3].
void launch_cgsr_init(cudaStream_t s, int n_own, const double* f, const uint8_t* fixed_mask, const double* dinv,
                      const double* binv, double* fbc, double* x, double* r, double* u, double* p, double* sv,
                      double* partial, CgState* st, int warm, const double* Kx0);
void launch_cgsr_update(cudaStream_t s, int n_own, const double* dinv, const double* binv, double* x, double* r,
                        double* u, const double* w, double* p, double* sv, double* partial, CgState* st,
                        int share = 1);
// The single-reduction update of every in-process part in one launch (grid.y = part).
struct SrPart {
  const double* dinv;
  const double* binv;
  double *x, *r, *u;
  const double* w;
  double *p, *sv, *partial;
  CgState* st;
  int n_own;
  int pad_;
};
void launch_cgsr_update_multi(cudaStream_t s, const SrPart* mp, int n_parts, int max_own);
void launch_cgsr_replace(cudaStream_t s, int n_own, const double* fbc, const double* Kx, const double* dinv,
                         const double* binv, double* r, double* u, double* partial, CgState* st);
// In-process halo fill of all parts in one launch: entry k = (dst part, dst node, src part,
// src node) copies the 6 values of a node between the parts' vectors base[part].
void launch_halo_gather(cudaStream_t s, int n_ent, const int4* ent, double* const* base);

// Lanczos certification (lanczos.cu): extreme Ritz values of M^-1 K from the recorded CG
// coefficients of every design (st->lz_min / lz_max; Tbuf scratch [B][cap][2]); the
// end-of-solve sums red[0..3] = |r|^2, r^T M^-1 r, f_bc^T x, x^T x of the true residual
// (binv != nullptr: node-block M); the per-design M scale (min 1/dinv or 1/|Binv_n|_F)
// as the bit pattern of a positive double, atomicMin-reduced into out[B] (pre-set to ~0).
void launch_lanczos_ritz(cudaStream_t s, CgState* st, double* Tbuf, int cap, int B);
void launch_cert_sums(cudaStream_t s, int n_nodes, const double* fbc, const double* Kx, const double* x,
                      const double* dinv, const double* binv, double* partial, CgState* st, const BatchStrides& bs);
void launch_mscale(cudaStream_t s, int n_nodes, const double* dinv, const double* binv, unsigned long long* out,
                   const BatchStrides& bs);
void launch_residual_norm(cudaStream_t s, int ndof, const double* f, const double* Kx,
                          double* partial, CgState* st,
    const BatchStrides& bs = BatchStrides());
void launch_zero_fixed(cudaStream_t s, int ndof, const uint8_t* fixed_mask, double* x,
    const BatchStrides& bs = BatchStrides());

// Partitioned-solve helpers
// Reliable updates (residual replacement): REPL_PERIODIC replaces r by f - K x for
// active designs whose r^T r fell below REPL_FACTOR * rr_ref; REPL_FINAL restarts
// (r = f - K x, p = z) converged designs whose TRUE residual exceeds 2 rtol.  Both
// only while |f - K x| <= REPL_DRIFT |r| (else the iterate has reached the fp64
// accuracy floor of K x and the design is marked `floor`: plain CG from then on).
enum ReplMode { REPL_PERIODIC = 0, REPL_FINAL = 1 };
constexpr double REPL_FACTOR = 1e-4;
constexpr int MAX_RESTARTS = 2;
constexpr double REPL_DRIFT = 10.0;
constexpr double REPL_CONT = 2.0;   // periodic replacement continues CG (beta from the replaced
                                    // r) while |f - K x| <= REPL_CONT |r|, else restarts (beta = 0)
void launch_cg_true_res(cudaStream_t s, int ndof, const double* fbc, const double* Kx, double* partial,
                        CgState* st, const BatchStrides& bs = BatchStrides());
void launch_cg_check(cudaStream_t s, CgState* st, int mode, int B);
void launch_cg_replace(cudaStream_t s, int ndof, const double* fbc, const double* Kx,
                       const double* dinv, double* r, double* p, double* partial, CgState* st, int mode,
                       const BatchStrides& bs = BatchStrides());
void launch_pack(cudaStream_t s, int count, const int32_t* idx, const double* vec, double* buf);
void launch_allreduce_parts(cudaStream_t s, CgState* const* sts, int n_parts, int nvals);
// out = a x + b y (elementwise, n doubles)
void launch_lincomb(cudaStream_t s, int64_t n, double a, const double* x, double b, const double* y, double* out);
void launch_gather(cudaStream_t s, int n, const int32_t* idx, const double* src, double* dst);
void launch_scatter(cudaStream_t s, int n, const int32_t* idx, const double* src, double* dst);
void launch_dot_local(cudaStream_t s, int n, const double* a, const double* b, double* partial,
                      CgState* st,
    const BatchStrides& bs = BatchStrides());

// Hat filter (filter.cu): points sorted by cell (px, py, pz, perm: sorted -> original),
// cell_of [2n]: sorted position of point i, then its cell id; cell_start [cells + 1].
void launch_hat_filter(cudaStream_t s, int n, int ncomp, const double* px, const double* py,
                       const double* pz, const int32_t* cell_of, const int32_t* perm,
                       const int64_t* cell_start, int gx, int gy, int gz, double radius,
                       const double* in, double* out);

// Design-dependent area loads (loads.cu): f += d (q + w t) A / 4 at the owned nodes; and
// slot_partial / dt += coef * v^T df/dp.
void launch_area_load(cudaStream_t s, int n_own, int n_beams, int n_quads, const double* x, const double* y,
                      const double* z, const int32_t* conn, const double* t, const double* lq, const double* lw,
                      const double dir[3], const int64_t* inc_ptr, const int32_t* inc_slot, double* a, double* f,
                      const BatchStrides& bs);
void launch_area_load_grad(cudaStream_t s, int n_beams, int n_quads, const double* x, const double* y,
                           const double* z, const int32_t* conn, const double* t, const double* lq,
                           const double* lw, const double dir[3], const double* v, double coef,
                           double* slot_partial, double* dt, const BatchStrides& bs);

// Gradient kernels
// SIMP density (grad.cu): E, G from rho^P and the reference moduli; dC/drho from dC/dE in place
void launch_simp_material(cudaStream_t s, int ne, const double* rho, double penal, const double* E0,
                          const double* G0, const double* nu, double* E, double* G);
void launch_simp_chain(cudaStream_t s, int ne, int B, const double* rho, double penal, const double* E0,
                       double* dE);
void launch_beam_grad(cudaStream_t s, int n_beams, const double* x, const double* y,
                      const double* z, const int32_t* conn, const double* A,
                      const double* Iy, const double* Iz, const double* J, const double* E,
                      const double* G, const double* u, double scale, double* slot_partial,
                      double* dC_dE, int n_elems, const BatchStrides& bs = BatchStrides(),
                      const double* v = nullptr);
// (v != nullptr: the bilinear -s d/dp [v_e^T K_e(p) u_e] instead of -s d/dp [u_e^T K_e u_e]:
// the general adjoint's -lambda^T dK/dp u in one pass)
void launch_quad_grad(cudaStream_t s, int n_beams, int n_quads, const double* x,
                      const double* y, const double* z, const int32_t* conn, const double* t,
                      const double* E, const double* nu, double drill_alpha, const double* u,
                      double scale, double* slot_partial, double* dC_dt, double* dC_dE,
                      const BatchStrides& bs = BatchStrides(), const double* v = nullptr);
void launch_node_reduce(cudaStream_t s, int n_nodes, const int64_t* inc_ptr,
                        const int32_t* inc_slot, const double* slot_partial, double* dC_dxyz,
    const BatchStrides& bs = BatchStrides());


extern long long g_launches;  // launch counter (per process; handles add their own deltas)

// After every launch: count it and report a launch-configuration error by name
// (the error stays pending for the caller's cudaGetLastError check).
#define SSO_POST_LAUNCH(name)                                                         \
  do {                                                                                \
    ++::sso::g_launches;                                                              \
    cudaError_t e__ = cudaPeekAtLastError();                                          \
    if (e__ != cudaSuccess) ::sso::note_launch_error(name, e__);                      \
  } while (0)
void note_launch_error(const char* name, cudaError_t e);
const char* last_launch_error();

// Cooperative launch (cudaLaunchAttributeCooperative) for the kernels with a grid-wide
// barrier: the driver guarantees that every CTA is co-resident or rejects the launch
// (cudaErrorCooperativeLaunchTooLarge) instead of leaving CTAs spinning on CTAs that
// cannot be scheduled (a shared GPU, MPS, concurrent streams).  Captures into graphs.
template <typename... K, typename... A>
inline cudaError_t launch_cooperative(void (*kern)(K...), dim3 grid, dim3 block, cudaStream_t s, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  static const bool coop = !(getenv("SSO_COOP") && getenv("SSO_COOP")[0] == '0');  // A/B switch
  cfg.attrs = at;
  cfg.numAttrs = coop ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}
#define SSO_POST_LAUNCH_RC(name, rc)                           \
  do {                                                         \
    ++::sso::g_launches;                                       \
    if ((rc) != cudaSuccess) ::sso::note_launch_error(name, rc); \
  } while (0)

}  // namespace sso

namespace sso {

// ---------------------------------------------------------------------------
// Partitioning: contiguous node ranges per part.  A part's
// local mesh = its owned nodes [begin, end) (local ids 0..n_own-1, global order)
// followed by its halo nodes (non-owned nodes of local elements) ordered by
// (owner part, global id).  Local elements = every element with at least one
// owned node, in ascending global order (so owned rows sum contributions in the
// same order as the global assembly: rank-local values are bit-identical).
// ---------------------------------------------------------------------------
struct NeighborPlan {
  int32_t part;                       // neighbour part / rank
  std::vector<int32_t> send_local;    // my owned local node ids it needs, in its halo order
  int32_t recv_offset = 0;            // first halo slot (relative to n_own) it fills
  int32_t recv_count = 0;
};

struct LocalMesh {
  int32_t part = 0, n_parts = 1;
  int32_t own_begin = 0, own_end = 0, n_own = 0;
  std::vector<int32_t> node_gid;      // local -> global node id
  std::vector<int32_t> beam_gid, quad_gid;   // local -> global element id (within type)
  std::vector<int32_t> beam_conn, quad_conn; // local numbering
  std::vector<int32_t> own_quad_local;       // local quads whose first node is owned
  std::vector<NeighborPlan> nbrs;
};

// ranges: [n_parts + 1] node boundaries (0 = ranges[0] < ... < ranges[n_parts] = n_nodes).
std::string build_local_mesh(int32_t n_nodes, int32_t n_beams, const int32_t* beam_conn,
                             int32_t n_quads, const int32_t* quad_conn, const int32_t* ranges,
                             int32_t n_parts, int32_t part, LocalMesh& L);

}  // namespace sso
