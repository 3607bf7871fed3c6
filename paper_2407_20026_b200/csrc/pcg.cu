// A3 — fp64 Jacobi-preconditioned CG kernels (sm_100a), SURVEY.md §8(a) A3.
//
// Solves K_bc u = f_bc (Eq. 1; supports by elimination, reading
// c1) with the CG of reading c10: x0 = 0, M = diag(K_bc), stop when
// |r|_2 <= rtol |f_bc|_2, breakdown p^T K p <= 0 -> NOT_SPD.
//
// Single-part handles (the default path), one iteration = 2 kernels, no host sync:
//   spmv_pull_cta_kernel   q = K p over the upper-block records (storage 3) and the
//                          per-CTA p^T q partials (left for the update: defer_alpha)
//   cg_update_fused_kernel every CTA sums the p^T q partials in one fixed order (alpha),
//                          x += alpha p, r -= alpha q, z = dinv r, r^T z, r^T r -> one
//                          all-CTA all-reduce (cg_fused.cuh; cooperative launch) -> beta,
//                          convergence test, p_next = z + beta p into the other p buffer
// (spmv_tma_kernel replaces the pull kernel with full storage; node-block Jacobi has its
// own fused update in block_jacobi.cu; partitioned handles run the single-reduction CG of
// cg_sr.cu).  The classic 3-kernel form (spmv_dot, cg_update, cg_pupdate) remains for
// SSO_CG_FUSED=0 and batches larger than the co-resident grid.  Every kernel returns
// immediately once `done` is set, so a fixed chunk of iterations is captured once in a CUDA
// graph and replayed; the host only polls `done` between chunks.  Reductions are
// atomic-free and in fixed order (per-CTA partials; last-CTA ticket reductions or the
// all-CTA all-reduce) -> bit-reproducible for a fixed grid.
//
// Full-storage layout (storage 1): the scalar CSR values of node n's six rows are contiguous
// at 36 node_ptr[n]; row 6n+a, column 6m+b with m = node_col[node_ptr[n]+k] sits at
// 36 node_ptr[n] + a (6 deg) + 6k + b; a warp streams each node's run through a shared
// memory ring and applies one x gather to all six rows.  Upper-block layout (storage 3,
// default): see the pull kernel below and DESIGN.md §5.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "cg_common.cuh"
#include "tma.cuh"
#include "cg_fused.cuh"
#include "sso_internal.h"

namespace sso {

long long g_launches = 0;
static char g_launch_err[256] = {0};
void note_launch_error(const char* name, cudaError_t e) {
  if (!g_launch_err[0]) snprintf(g_launch_err, sizeof g_launch_err, "%s: %s", name, cudaGetErrorString(e));
}
const char* last_launch_error() { return g_launch_err; }

namespace {

int g_sms = 0;

// Transposed butterfly: reduce 6 (padded to 8) per-lane values across the warp
// in 9 shuffles.  On return, lane L holds the total of value index
// vi(L) = 4 bit4(L) + 2 bit3(L) + bit2(L) (valid for every L; lanes sharing vi agree).
__device__ __forceinline__ double reduce6(double (&acc)[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double send = b4 ? acc[k] : acc[k + 4];
    double keep = b4 ? acc[k + 4] : acc[k];
    acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    double send = b3 ? acc[k] : acc[k + 2];
    double keep = b3 ? acc[k + 2] : acc[k];
    acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    double send = b2 ? acc[0] : acc[1];
    double keep = b2 ? acc[1] : acc[0];
    acc[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 2);
  acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
  return acc[0];
}

// ---------------------------------------------------------------------------
// TMA-pipelined node-block SpMV, warp-independent.
//
// Every warp owns a contiguous range of nodes.  The six rows of a node are ONE
// contiguous run of 36 deg values, so lane 0 of the warp streams the runs of
// its next nodes into a private ring of SPMV_STAGES shared-memory slots with
// cp.async.bulk (TMA bulk copy, completion on a per-slot mbarrier, L2
// evict-first so the CG vectors stay L2-resident) while the warp computes the
// current node.  Warps never wait for each other.  Per node the warp gathers
// p[6m+b] once per row position (m from a register copy of the node's column
// list, via shuffle; prefetched one node ahead) and applies it to the six
// rows; a 9-shuffle transposed butterfly reduces the six row sums.  A node
// whose run exceeds a slot (degree > SLOT_DEG) is read from global memory.
// ---------------------------------------------------------------------------
constexpr int SPMV_WARPS = 8;

// Six row sums of a node whose 36 deg values start at `base` (shared or global);
// ncol = node_col[b0 + lane] for lane < deg (deg <= 32), else read from node_col.
// Returns y[6n + vi(lane)] in every lane.
__device__ __forceinline__ double node_rows(const double* base, int64_t b0, int deg, int ncol,
                                            const int32_t* __restrict__ node_col,
                                            const double* __restrict__ x, int lane) {
  const int rowlen = 6 * deg;
  double acc[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) acc[a] = 0.0;
  if (deg <= 32) {
    // two adjacent row positions per lane (same 6x6 block: positions are even and 6
    // is even): 128-bit shared loads of the values and one 128-bit gather of x
    for (int r0 = 0; r0 < rowlen; r0 += 64) {
      const int ra = r0 + 2 * lane;
      const bool aa = ra < rowlen;
      const int ka = aa ? ra / 6 : 0;
      const int ma = __shfl_sync(0xffffffffu, ncol, ka);
      double2 xv = make_double2(0.0, 0.0);
      if (aa) xv = *reinterpret_cast<const double2*>(x + 6 * (int64_t)ma + (ra - 6 * ka));
      if (aa) {
#pragma unroll
        for (int a = 0; a < 6; ++a) {
          const double2 v = *reinterpret_cast<const double2*>(base + a * rowlen + ra);
          acc[a] = fma(v.y, xv.y, fma(v.x, xv.x, acc[a]));
        }
      }
    }
  } else {
    for (int rem = lane; rem < rowlen; rem += 32) {
      const int k = rem / 6;
      const int m = __ldg(node_col + b0 + k);
      const double xv = x[6 * (int64_t)m + (rem - 6 * k)];
#pragma unroll
      for (int a = 0; a < 6; ++a) acc[a] += base[a * rowlen + rem] * xv;
    }
  }
  return reduce6(acc, lane);
}

// ---------------------------------------------------------------------------
// Symmetric (upper-block) storage SpMV.  Pass 1, warp-independent TMA rings as
// above, two nodes per step: for node n the upper row sums y_n = sum_{m >= n}
// K_nm x_m, and per off-diagonal upper block the transpose contribution
// t = K_nm^T x_n written to its receiver-ordered slot.  In the CG form (DOT) the
// same values give p^T K p = sum_n (2 p_n . y_n - p_n^T K_nn p_n): the diagonal
// term is sum over the lanes holding block 0 of t_b p_n[b], so alpha is formed
// at the end of pass 1 and the receiver sums move into the x / r update.
// ---------------------------------------------------------------------------

// q = K p; with DOT also p^T q -> alpha (CG) and an early exit once `done`.
// STAGES ring slots of SLOT_DEG 6x6 blocks per warp; MINB CTAs per SM.
template <bool DOT, int SPMV_STAGES, int SLOT_DEG, int MINB>
__global__ void __launch_bounds__(SPMV_WARPS * 32, MINB) spmv_tma_kernel(
    int n_nodes, int nodes_per_warp, const int64_t* __restrict__ node_ptr,
    const int32_t* __restrict__ node_col, const double* __restrict__ vals,
    const double* __restrict__ p, double* __restrict__ q, double* __restrict__ partial,
    CgState* st, BatchStrides bs) {
  constexpr int SLOT_DOUBLES = 36 * SLOT_DEG;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar[SPMV_WARPS][SPMV_STAGES];
  __shared__ double sm[32];
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    vals += bd * bs.nnz;
    p += bd * bs.dof;
    q += bd * bs.dof;
    if (DOT) {
      partial += bd * bs.partial;
      st += bd;
    }
  }
  if (DOT && st->done) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t gw = (int64_t)blockIdx.x * SPMV_WARPS + warp;
  const int64_t nb = gw * nodes_per_warp;
  const int64_t left = (int64_t)n_nodes - nb;
  const int cnt = left <= 0 ? 0 : (int)(left < nodes_per_warp ? left : nodes_per_warp);
  double* ring = reinterpret_cast<double*>(smem_raw) + (size_t)warp * SPMV_STAGES * SLOT_DOUBLES;
  uint64_t* wbar = bar[warp];
  uint64_t pol = 0;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < SPMV_STAGES; ++s) mbar_init(&wbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pol = evict_first_policy();
  }
  __syncwarp();
  auto issue = [&](int k) {  // lane 0 only
    const int64_t n = nb + k;
    const int s = k % SPMV_STAGES;
    const int64_t b0 = node_ptr[n], b1 = node_ptr[n + 1];
    if (b1 - b0 <= SLOT_DEG) {
      const unsigned bytes = (unsigned)(288 * (b1 - b0));
      mbar_arrive_expect_tx(&wbar[s], bytes);
      bulk_g2s(ring + (size_t)s * SLOT_DOUBLES, vals + 36 * b0, bytes, &wbar[s], pol);
    } else {
      mbar_arrive(&wbar[s]);  // oversized node: read from global, keep the phase sequence
    }
  };
  if (lane == 0)
    for (int k = 0; k < min(SPMV_STAGES - 1, cnt); ++k) issue(k);
  const int vi = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  const bool writer = ((lane & 3) == 0) && vi < 6;
  double pq[1] = {0.0};
  // metadata of the current node, prefetched one node ahead
  int64_t b0n = 0;
  int degn = 0, ncoln = 0;
  if (cnt > 0) {
    b0n = node_ptr[nb];
    degn = (int)(node_ptr[nb + 1] - b0n);
    ncoln = (lane < degn) ? __ldg(node_col + b0n + lane) : 0;
  }
  for (int k = 0; k < cnt; ++k) {
    const int s = k % SPMV_STAGES;
    if (lane == 0 && k + SPMV_STAGES - 1 < cnt) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + SPMV_STAGES - 1);
    }
    const int64_t n = nb + k;
    const int64_t b0 = b0n;
    const int deg = degn, ncol = ncoln;
    if (k + 1 < cnt) {
      b0n = node_ptr[n + 1];
      degn = (int)(node_ptr[n + 2] - b0n);
      ncoln = (lane < degn) ? __ldg(node_col + b0n + lane) : 0;
    }
    mbar_wait(&wbar[s], (unsigned)((k / SPMV_STAGES) & 1));
    const double* base = (deg <= SLOT_DEG) ? ring + (size_t)s * SLOT_DOUBLES : vals + 36 * b0;
    const double y = node_rows(base, b0, deg, ncol, node_col, p, lane);
    if (writer) {
      q[6 * n + vi] = y;
      if (DOT) pq[0] += p[6 * n + vi] * y;
    }
    __syncwarp();
  }
  if (DOT) {
    if (st->defer_alpha) {  // the fused update sums the partials (fixed order) in every CTA
      block_sum<1>(pq, sm);
      if (threadIdx.x == 0) {
        partial[PQ_OFF + blockIdx.x] = pq[0];
        if (blockIdx.x == 0) st->npq = (int)gridDim.x;
      }
    } else if (grid_sum<1>(pq, partial, &st->ticket[0], sm) && threadIdx.x == 0) {
      if (st->dist) {
        st->red[0] = pq[0];
        return;
      }
      st->pq = pq[0];
      if (!(pq[0] > 0.0)) {
        st->status = SSO_E_NOT_SPD;
        st->done = 1;
      } else {
        st->alpha = st->rz / pq[0];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Symmetric "pull" SpMV (storage 3).  Only the upper node blocks (n, m >= n) are
// stored.  Each block is one contiguous record of PULL_BLOCK = 38 doubles: nine 2x2
// sub-blocks of 4 doubles (column-major inside; rec_off in sso_internal.h) followed by
// 2 zero pad doubles.  The pad makes the record stride 19 16-byte words (odd), which
// spreads the 16-byte shared-memory reads of the consumers over all bank groups (an
// 18-word stride keeps them on even groups: 2-way conflicts).  The 2x2 sub-blocks let one
// instruction sequence serve both uses of a block (K_mj x_j for its row node, K_nm^T x_n
// for its column node) with no divergent branch.  A node's upper run is its records
// for k = 0 .. udeg-1 (block k at PULL_BLOCK (uptr[n] + k)).  The row node m needs
//   y_m = sum_{j >= m} K_mj x_j + sum_{n < m} K_nm^T x_n:
// its own run (contiguous) and the records (n, m) of its lower neighbours n < m,
// formed in one pass with no transpose buffer, no atomics and a fixed order.
// Nodes are processed in round-robin chunks, so at any time the GPU works on one
// window of consecutive nodes and a pulled record was streamed by its owner (or is
// about to be) within that window -- an L2 hit: DRAM sees each stored value once
// (~0.56 of the full-storage bytes on shell grids).
// ---------------------------------------------------------------------------
// Per-node pull descriptor (16 int32, built on the host, SSO pattern order):
//   d[0] = first upper block of the node (its run starts at PULL_BLOCK d[0]),
//   d[1] = udeg | ldeg << 8 | fits << 16,
//   fits:  d[2 .. 2+udeg) upper block columns, then (source node, upper block) of each
//          pulled block at d[2+udeg+2j], d[3+udeg+2j];
//   !fits: d[2] = first pull-list entry (lptr) -- the node takes the general path.
// A node fits when udeg <= PULL_MAX_UDEG and ldeg <= 4: its pulled records come with
// ONE TMA tile::gather4 of 4 rows of the [blocks][PULL_BLOCK] view of the values
// (padding rows repeat the node's own first block).
constexpr int PULL_DESC = 16;
constexpr int PULL_MAX_UDEG = 5;

__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int r0, int r1, int r2, int r3,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "l"(policy)
      : "memory");
}

// ---------------------------------------------------------------------------
// Pull SpMV, warp-specialised chunk form (storage 3, the default pull kernel).
// The per-node bookkeeping that made the warp-per-node form issue-bound (descriptor
// shuffles, two TMA issues per node) is done lane-parallel by a PRODUCER warp: a
// CTA takes chunks of C consecutive nodes (chunks dealt round-robin over the CTAs,
// so the GPU sweeps one window of nodes and pulled blocks stay L2 hits); producer
// lane i loads node i's descriptor into shared memory and issues that node's
// gather4 of pulled blocks, lane 0 issues ONE bulk copy of the chunk's own upper
// runs (consecutive nodes' runs are contiguous).  NB buffers with full / empty
// mbarriers; W CONSUMER warps each take C / W nodes of
// a chunk with no CTA-wide barrier: lane 3j + h forms (t_2h, t_2h+1) of block j
// (own upper blocks, then pulled) as in the warp form, a per-warp shared row sums
// them in ascending j.  Chunks holding a node that does not fit (udeg > 5 or
// ldeg > 4) take a general path reading the values from global memory.
// ---------------------------------------------------------------------------
// Consumer lane -> compute unit u = 3 j + h (31 = idle).  Checked by tests/test_pull_layout.py
// against the shared-memory bank model of tools/pull_lane_perm.py for the 2x2 sub-block
// records (19-word record stride, own region after the 80-word pulled slots): 34/7 = 4.86
// wavefronts per 16-byte load of an interior node (the identity needs 6.5), the optimum of
// an annealing search over lane and sub-block slot permutations (tools/pull_perm_anneal.c),
// and the three lanes of a block (same 48-byte x gather) share a quarter warp for all
// blocks but one.
__constant__ int8_t kPullUnitOfLane[32] = {15, 31, 18, 20, 17, 16, 31, 19, 25, 23, 26, 22, 31, 24, 31, 21,
                                           3, 7, 9, 4, 5, 8, 6, 10, 14, 13, 2, 12, 1, 11, 0, 31};

template <int C, int W>
struct PullChunkSmem {
  static constexpr int PSLOT = 160;                // doubles per node: 4 gathered records (1216 B) -> 1280 B
  static constexpr int PULL = PSLOT * C;           // doubles: pulled records (128-byte aligned per node)
  static constexpr int OWN = PULL_BLOCK * 5 * C;   // doubles: own upper runs (<= 5 blocks per node)
  static constexpr int DESC = PULL_DESC * C / 2;   // doubles holding the C descriptors (16 int32 each)
  static constexpr int BUF = (PULL + OWN + DESC + 15) / 16 * 16;  // per buffer, 128-byte multiple
                                                                   // (PULL first: aligned gather4 rows)
  static constexpr int NPW = C / W;                // nodes per consumer warp per chunk
  static constexpr int RED = 2 * 27 * NPW;         // doubles per consumer warp
};

template <bool DOT, int C, int NB, int MINB, int W>
__global__ void __launch_bounds__(32 * (W + 1), MINB) spmv_pull_cta_kernel(
    const __grid_constant__ CUtensorMap tmap, int n_nodes, int node0, int red_add, int rows_per_design,
    const int32_t* __restrict__ pdesc,
    const int32_t* __restrict__ ucol, const int2* __restrict__ lpull, const double* __restrict__ vals,
    const double* __restrict__ p, double* __restrict__ q, double* __restrict__ partial, CgState* st,
    BatchStrides bs, const PullPart* __restrict__ mp) {
  using S = PullChunkSmem<C, W>;
  constexpr int NPW = S::NPW;
  constexpr unsigned FULL = 0xffffffffu;
  static_assert(C <= 32 && C % W == 0, "chunk size");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[NB];   // chunk data landed (bulk copy + gathers)
  __shared__ __align__(8) uint64_t desc_bar[NB];   // chunk descriptors written (x gathers may start)
  __shared__ __align__(8) uint64_t empty_bar[NB];  // consumers done with the buffer
  __shared__ int chunk_fits[NB];
  __shared__ double sm[32];
  int row0 = blockIdx.y * rows_per_design;
  const CUtensorMap* tm = &tmap;
  if (mp) {  // part blockIdx.y of a multi-part launch: its own operands and tensor map
    const PullPart& A = mp[blockIdx.y];
    tm = &A.tmap;
    row0 = 0;
    n_nodes = A.n_nodes;
    pdesc = A.pdesc;
    ucol = A.ucol;
    lpull = A.lpull;
    vals = A.vals;
    p = A.x;
    q = A.y;
    if (DOT) {
      partial = A.partial;
      st = A.st;
    }
  } else {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    vals += bd * bs.nnz;
    p += bd * bs.dof;
    q += bd * bs.dof;
    if (DOT) {
      partial += bd * bs.partial;
      st += bd;
    }
  }
  if (DOT && st->done) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // rows [node0, n_nodes): the whole owned range, or one piece of it (partitioned handles
  // overlap the halo exchange with the rows that need no halo values)
  const int n_chunks = (n_nodes - node0 + C - 1) / C;
  const int cnt = (int)blockIdx.x < n_chunks ? (n_chunks - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  double* sbase = reinterpret_cast<double*>(smem_raw);
  double* red_base = sbase + (size_t)NB * S::BUF;
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full_bar[b], 1);
      mbar_init(&desc_bar[b], 1);
      mbar_init(&empty_bar[b], W);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double pq[1] = {0.0};
  if (warp == W) {
    // ---------------- producer ----------------
    // evict-first: a record is pulled again (by its column node) by a chunk of the same window
    // soon after; parts launched together stretch that distance, so they keep records
    // evict-normal (C4 in 8 strips: 516 -> 505 us per iteration; a single C3b part loses its
    // L2-resident CG vectors with evict-normal: 68.9 -> 76.1 us)
    const uint64_t pol = mp ? evict_normal_policy() : evict_first_policy();
    // descriptors of chunk k are loaded one chunk ahead (off the empty-barrier critical path)
    auto load_desc = [&](int k, int4& a, int4& b2, int4& c, int4& d) {
      const int first = node0 + ((int)blockIdx.x + k * (int)gridDim.x) * C;
      a = b2 = c = d = make_int4(0, 0, 0, 0);
      if (k < cnt && lane < min(C, n_nodes - first)) {
        const int4* src = reinterpret_cast<const int4*>(pdesc + PULL_DESC * ((int64_t)first + lane));
        a = __ldg(src);
        b2 = __ldg(src + 1);
        c = __ldg(src + 2);
        d = __ldg(src + 3);
      }
    };
    int4 n0, n1, n2, n3;
    load_desc(0, n0, n1, n2, n3);
    for (int k = 0; k < cnt; ++k) {
      const int b = k % NB;
      const int4 d0 = n0, d1 = n1, d2 = n2, d3 = n3;
      load_desc(k + 1, n0, n1, n2, n3);
      if (k >= NB) mbar_wait(&empty_bar[b], (unsigned)(((k / NB) - 1) & 1));
      double* buf = sbase + (size_t)b * S::BUF;
      int32_t* D = reinterpret_cast<int32_t*>(buf + S::PULL + S::OWN);
      const int first = node0 + ((int)blockIdx.x + k * (int)gridDim.x) * C;
      const int nc = min(C, n_nodes - first);
      if (lane < nc) {
        int4* dst = reinterpret_cast<int4*>(D + PULL_DESC * lane);
        dst[0] = d0;
        dst[1] = d1;
        dst[2] = d2;
        dst[3] = d3;
      }
      const int fl = d0.y;
      const int udeg = fl & 255, ldeg = (fl >> 8) & 255;
      const bool all_fit = __all_sync(FULL, lane >= nc || ((fl >> 16) & 1));
      const unsigned has_pull = __ballot_sync(FULL, lane < nc && ldeg > 0);
      const int b_first = __shfl_sync(FULL, d0.x, 0);
      const int b_end = __shfl_sync(FULL, d0.x + udeg, nc - 1);
      // generic reads of buffer b by the consumers of chunk k - NB precede the async writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        chunk_fits[b] = all_fit ? 1 : 0;
        mbar_arrive(&desc_bar[b]);  // release: descriptors and the fit flag are visible
        if (all_fit) {
          mbar_arrive_expect_tx(&full_bar[b],
                                (unsigned)(8 * PULL_BLOCK * (b_end - b_first + 4 * __popc(has_pull))));
          bulk_g2s(buf + S::PULL, vals + PULL_BLOCK * (int64_t)b_first, (unsigned)(8 * PULL_BLOCK * (b_end - b_first)),
                   &full_bar[b], pol);
        } else {
          mbar_arrive(&full_bar[b]);  // release: the descriptors written above are visible
        }
      }
      __syncwarp();  // expect_tx registered before the gathers complete
      if (all_fit && lane < nc && ldeg > 0) {
        // pulled block i of the node: (source, block) at d[2 + udeg + 2i] (re-read from this lane's
        // own shared-memory copy of the descriptor); pad with the own first block
        const int32_t* Dl = D + PULL_DESC * lane + 3 + udeg;
        int r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) r[i] = row0 + (i < ldeg ? Dl[2 * i] : d0.x);
        tma_gather4(buf + S::PSLOT * lane, tm, r[0], r[1], r[2], r[3], &full_bar[b], pol);
      }
    }
  } else {
    // ---------------- consumers ----------------
    double2* red = reinterpret_cast<double2*>(red_base) + (size_t)warp * 27 * NPW;
    const int ul = kPullUnitOfLane[lane];
    const int jl = ul < 27 ? ul / 3 : 9, hl = ul < 27 ? ul - 3 * (ul / 3) : 0;
    // this lane's sub-block offsets inside a record: own units (h, sb), pulled units (sb, h)
    int offO[3], offP[3];
#pragma unroll
    for (int sb = 0; sb < 3; ++sb) {
      offO[sb] = pull_sub_off(3 * sb + hl);
      offP[sb] = pull_sub_off(3 * hl + sb);
    }
    for (int k = 0; k < cnt; ++k) {
      const int b = k % NB;
      const double* buf = sbase + (size_t)b * S::BUF;
      const double* own = buf + S::PULL;
      const int32_t* D = reinterpret_cast<const int32_t*>(buf + S::PULL + S::OWN);
      const int first = node0 + ((int)blockIdx.x + k * (int)gridDim.x) * C;
      const int nc = min(C, n_nodes - first);
      mbar_wait(&desc_bar[b], (unsigned)((k / NB) & 1));
      if (chunk_fits[b]) {
        const int b_first = D[0];
        const double* blk[NPW];
        double2 xv[NPW][3];
        bool act[NPW], ownb[NPW];
#pragma unroll
        for (int e = 0; e < NPW; ++e) {  // node i = warp + 8 e of the chunk: operands first
          const int i = warp + W * e;
          const int* Di = D + PULL_DESC * (i < nc ? i : 0);
          const int fl = Di[1];
          const int udeg = fl & 255, nb = udeg + ((fl >> 8) & 255);
          act[e] = i < nc && jl < nb;
          blk[e] = own;
          ownb[e] = jl < udeg;
          if (act[e]) {
            int xn;
            if (jl < udeg) {
              blk[e] = own + PULL_BLOCK * (Di[0] - b_first + jl);
              xn = Di[2 + jl];
            } else {
              blk[e] = buf + S::PSLOT * i + PULL_BLOCK * (jl - udeg);
              xn = Di[2 + 2 * jl - udeg];
            }
            const double2* xp = reinterpret_cast<const double2*>(p + 6 * (int64_t)xn);
            xv[e][0] = xp[0];
            xv[e][1] = xp[1];
            xv[e][2] = xp[2];
          }
        }
        // p of this lane's output row (p^T q), loaded with the x gathers
        double prow = 0.0;
        if (DOT && lane < 6 * NPW) {
          const int e = lane / 6, a = lane - 6 * e;
          const int i = warp + W * e;
          if (i < nc) prow = p[6 * ((int64_t)first + i) + a];
        }
        mbar_wait(&full_bar[b], (unsigned)((k / NB) & 1));  // x gathers overlap the chunk's data
#pragma unroll
        for (int e = 0; e < NPW; ++e) {
          if (ul >= 27) continue;
          // inactive units (j beyond the node's blocks) write zeros: the row sums below add all
          // nine entries in a fixed tree
          double t0 = 0.0, t1 = 0.0;
          if (act[e]) {
            // Branch-free over own and pulled units.  Sub-block k = (k00, k10 | k01, k11) of the
            // unit's strip: own K_mj uses sub-blocks (h, sb) -- outputs 2h, 2h+1 = rows, x_j
            // components 2 sb, 2 sb + 1 = columns; pulled K_nm^T uses (sb, h) -- outputs =
            // columns of K, x_n components = rows.  Both are t0 += k00 X0 + m X1,
            // t1 += n X0 + k11 X1 with (m, n) = (k01, k10) own, (k10, k01) pulled; even and odd
            // components in separate chains (the summation order of the oracle-checked form).
            const bool ow = ownb[e];
            double2 P[3], Q[3];
#pragma unroll
            for (int sb = 0; sb < 3; ++sb) {
              const double* sp = blk[e] + (ow ? offO[sb] : offP[sb]);
              P[sb] = *reinterpret_cast<const double2*>(sp);
              Q[sb] = *reinterpret_cast<const double2*>(sp + 2);
            }
            double m[3], n[3];
#pragma unroll
            for (int sb = 0; sb < 3; ++sb) {
              m[sb] = ow ? Q[sb].x : P[sb].y;
              n[sb] = ow ? P[sb].y : Q[sb].x;
            }
            const double2 x0 = xv[e][0], x1 = xv[e][1], x2 = xv[e][2];
            double u0, u1;
            t0 = P[0].x * x0.x;
            t1 = n[0] * x0.x;
            u0 = m[0] * x0.y;
            u1 = Q[0].y * x0.y;
            t0 = fma(P[1].x, x1.x, t0);
            t1 = fma(n[1], x1.x, t1);
            u0 = fma(m[1], x1.y, u0);
            u1 = fma(Q[1].y, x1.y, u1);
            t0 = fma(P[2].x, x2.x, t0);
            t1 = fma(n[2], x2.x, t1);
            u0 = fma(m[2], x2.y, u0);
            u1 = fma(Q[2].y, x2.y, u1);
            t0 += u0;
            t1 += u1;
          }
          red[27 * e + ul] = make_double2(t0, t1);
        }
        __syncwarp();
        // lane 6 e + a (< 6 NPW): row a of node e, the nine block entries in a fixed tree
        if (lane < 6 * NPW) {
          const int e = lane / 6, a = lane - 6 * e;
          const int i = warp + W * e;
          if (i < nc) {
            const double* rd = reinterpret_cast<const double*>(red + 27 * e) + a;
            double r9[9];
#pragma unroll
            for (int j = 0; j < 9; ++j) r9[j] = rd[6 * j];
            const double y = (((r9[0] + r9[1]) + (r9[2] + r9[3])) + ((r9[4] + r9[5]) + (r9[6] + r9[7]))) + r9[8];
            const int64_t row = 6 * ((int64_t)first + i) + a;
            q[row] = y;
            if (DOT) pq[0] += prow * y;
          }
        }
      } else if (lane < 6 * NPW) {
        mbar_wait(&full_bar[b], (unsigned)((k / NB) & 1));  // (no data: keeps the phase sequence)
        // general chunk: lane (node e, row a) sums its row from global memory, own blocks then
        // pulled blocks in ascending order (the order of the fast path)
        const int e = lane / 6, a = lane - 6 * e;
        const int i = warp + W * e;
        if (i < nc) {
          const int* Di = D + PULL_DESC * i;
          const int b0 = Di[0], fl = Di[1];
          const int udeg = fl & 255, ldeg = (fl >> 8) & 255;
          const bool fitn = (fl >> 16) & 1;
          const int l0 = fitn ? 0 : Di[2];
          double y = 0.0;
          for (int kb = 0; kb < udeg; ++kb) {
            const int m = fitn ? Di[2 + kb] : __ldg(ucol + b0 + kb);
            const double* bk = vals + PULL_BLOCK * ((int64_t)b0 + kb);
            double t = 0.0;
#pragma unroll
            for (int c = 0; c < 6; ++c) t = fma(bk[rec_off(a, c)], p[6 * (int64_t)m + c], t);
            y += t;
          }
          for (int jp = 0; jp < ldeg; ++jp) {
            const int2 e2 = fitn ? make_int2(Di[2 + udeg + 2 * jp], Di[3 + udeg + 2 * jp]) : __ldg(lpull + l0 + jp);
            const double* bk = vals + PULL_BLOCK * (int64_t)e2.y;
            double t = 0.0;
#pragma unroll
            for (int c = 0; c < 6; ++c) t = fma(bk[rec_off(c, a)], p[6 * (int64_t)e2.x + c], t);
            y += t;
          }
          const int64_t row = 6 * ((int64_t)first + i) + a;
          q[row] = y;
          if (DOT) pq[0] += p[row] * y;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[b]);  // this warp is done with buffer b
    }
  }
  if (DOT) {
    if (st->defer_alpha) {  // the fused update sums the partials (fixed order) in every CTA
      block_sum<1>(pq, sm);
      if (threadIdx.x == 0) {
        partial[PQ_OFF + blockIdx.x] = pq[0];
        if (blockIdx.x == 0) st->npq = (int)gridDim.x;
      }
    } else if (grid_sum<1>(pq, partial, &st->ticket[0], sm) && threadIdx.x == 0) {
      if (st->dist) {
        st->red[0] = (red_add ? st->red[0] : 0.0) + pq[0];  // pieces add in launch order
        return;
      }
      st->pq = pq[0];
      if (!(pq[0] > 0.0)) {
        st->status = SSO_E_NOT_SPD;
        st->done = 1;
      } else {
        st->alpha = st->rz / pq[0];
      }
    }
  }
}

// x += alpha p, r -= alpha q, z = dinv r; partial r^T z, r^T r.  double2 streams
// (ndof = 6 n is even; cudaMalloc buffers are 256 B aligned).
__global__ void __launch_bounds__(256) cg_update_kernel(int ndof, const double* __restrict__ dinv,
                                                        double* __restrict__ x,
                                                        double* __restrict__ r,
                                                        const double* __restrict__ p,
                                                        const double* __restrict__ q,
                                                        double* __restrict__ partial,
                                                        CgState* st, BatchStrides bs) {
  __shared__ double sm[64];
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    dinv += bd * bs.dof;
    x += bd * bs.dof;
    r += bd * bs.dof;
    p += bd * bs.dof;
    q += bd * bs.dof;
    partial += bd * bs.partial;
    st += bd;
  }
  if (st->done) return;
  const double alpha = st->alpha;
  double v[2] = {0.0, 0.0};  // r^T z, r^T r
  const int64_t n2 = ndof / 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double2* __restrict__ p2 = reinterpret_cast<const double2*>(p);
  const double2* __restrict__ q2 = reinterpret_cast<const double2*>(q);
  const double2* __restrict__ d2 = reinterpret_cast<const double2*>(dinv);
  double2* __restrict__ x2 = reinterpret_cast<double2*>(x);
  double2* __restrict__ r2 = reinterpret_cast<double2*>(r);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    const double2 pi = p2[i], qi = q2[i], di = d2[i];
    double2 xi = x2[i], ri = r2[i];
    xi.x += alpha * pi.x;
    xi.y += alpha * pi.y;
    ri.x -= alpha * qi.x;
    ri.y -= alpha * qi.y;
    x2[i] = xi;
    r2[i] = ri;
    v[0] += ri.x * (di.x * ri.x) + ri.y * (di.y * ri.y);
    v[1] += ri.x * ri.x + ri.y * ri.y;
  }
  if (grid_sum<2>(v, partial, &st->ticket[1], sm) && threadIdx.x == 0) {
    const double rz_new = v[0];
    st->beta = rz_new / st->rz;
    st->rz_prev = st->rz;
    st->rz = rz_new;
    st->rr = v[1];
    st->iter += 1;
    lz_record(st, st->alpha, st->beta);
    if (v[1] <= st->tol2) {
      st->done = 1;
      st->status = SSO_OK;
    } else if (st->iter >= st->max_iter) {
      st->done = 1;
      st->status = SSO_E_NOT_CONVERGED;
    }
  }
}

__global__ void __launch_bounds__(256) cg_pupdate_kernel(int ndof, const double* __restrict__ dinv,
                                                         const double* __restrict__ r,
                                                         double* __restrict__ p,
                                                         const CgState* st, BatchStrides bs) {
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    dinv += bd * bs.dof;
    r += bd * bs.dof;
    p += bd * bs.dof;
    st += bd;
  }
  if (st->done) return;
  const double beta = st->beta;
  const int64_t n2 = ndof / 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double2* __restrict__ r2 = reinterpret_cast<const double2*>(r);
  const double2* __restrict__ d2 = reinterpret_cast<const double2*>(dinv);
  double2* __restrict__ p2 = reinterpret_cast<double2*>(p);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    const double2 ri = r2[i], di = d2[i];
    double2 pi = p2[i];
    // z = dinv r rounded, then one fma: the rounding of cg_update_fused_kernel
    pi.x = __fma_rn(beta, pi.x, __dmul_rn(di.x, ri.x));
    pi.y = __fma_rn(beta, pi.y, __dmul_rn(di.y, ri.y));
    p2[i] = pi;
  }
}

// Fused form of cg_update + cg_pupdate for the designs of one part (point Jacobi).
// Phase 1 as cg_update_kernel (x += alpha p, r -= alpha q, z = dinv r; r^T z, r^T r
// over the grid, the last CTA forms beta and the convergence test); then a grid-wide
// barrier (cg_fused.cuh) and phase 2: p_next = z + beta p, from registers for the
// first FUSED_ITEMS double2 of each thread.  p_next goes to the OTHER p buffer
// (ping-pong), so a residual replacement can re-form it (cg_pfix).
constexpr int FUSED_ITEMS = 7;

__global__ void __launch_bounds__(256, 2) cg_update_fused_kernel(int ndof, const double* __restrict__ dinv,
                                                                 double* __restrict__ x,
                                                                 double* __restrict__ r,
                                                                 const double* __restrict__ p,
                                                                 const double* __restrict__ q,
                                                                 double* __restrict__ pn,
                                                                 double* __restrict__ partial,
                                                                 CgState* st, BatchStrides bs) {
  __shared__ double sm[64];
  {  // design of a batch (blockIdx.y): its own CTAs, reduction and barrier
    const int bd = blockIdx.y;
    dinv += bd * bs.dof;
    x += bd * bs.dof;
    r += bd * bs.dof;
    p += bd * bs.dof;
    q += bd * bs.dof;
    pn += bd * bs.dof;
    partial += bd * bs.partial;
    st += bd;
  }
  if (st->done) return;  // set only by earlier kernels: the same for every CTA
  // read before the all-reduce (CTA 0 rewrites them after every CTA has arrived)
  const double rz_old = st->rz;
  const long long iter_old = st->iter;
  double alpha, pqv;
  if (!cg_fused_alpha(partial + PQ_OFF, st, sm, rz_old, alpha, pqv)) return;
  double v[2] = {0.0, 0.0};  // r^T z, r^T r
  const int64_t n2 = ndof / 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double2* __restrict__ p2 = reinterpret_cast<const double2*>(p);
  const double2* __restrict__ q2 = reinterpret_cast<const double2*>(q);
  const double2* __restrict__ d2 = reinterpret_cast<const double2*>(dinv);
  double2* __restrict__ x2 = reinterpret_cast<double2*>(x);
  double2* __restrict__ r2 = reinterpret_cast<double2*>(r);
  double2* __restrict__ pn2 = reinterpret_cast<double2*>(pn);
  double2 zk[FUSED_ITEMS], pk[FUSED_ITEMS];
#pragma unroll
  for (int k = 0; k < FUSED_ITEMS; ++k) {
    const int64_t i = i0 + k * stride;
    zk[k] = pk[k] = make_double2(0.0, 0.0);
    if (i < n2) {
      const double2 pi = p2[i], qi = q2[i], di = d2[i];
      double2 xi = x2[i], ri = r2[i];
      xi.x += alpha * pi.x;
      xi.y += alpha * pi.y;
      ri.x -= alpha * qi.x;
      ri.y -= alpha * qi.y;
      x2[i] = xi;
      r2[i] = ri;
      v[0] += ri.x * (di.x * ri.x) + ri.y * (di.y * ri.y);
      v[1] += ri.x * ri.x + ri.y * ri.y;
      zk[k] = make_double2(__dmul_rn(di.x, ri.x), __dmul_rn(di.y, ri.y));
      pk[k] = pi;
    }
  }
  for (int64_t i = i0 + FUSED_ITEMS * stride; i < n2; i += stride) {
    const double2 pi = p2[i], qi = q2[i], di = d2[i];
    double2 xi = x2[i], ri = r2[i];
    xi.x += alpha * pi.x;
    xi.y += alpha * pi.y;
    ri.x -= alpha * qi.x;
    ri.y -= alpha * qi.y;
    x2[i] = xi;
    r2[i] = ri;
    v[0] += ri.x * (di.x * ri.x) + ri.y * (di.y * ri.y);
    v[1] += ri.x * ri.x + ri.y * ri.y;
  }
  if (!cg_fused_allreduce(v, partial, &st->arrive, sm)) {
    if (threadIdx.x == 0) {
      st->status = SSO_E_CUDA;
      st->done = 1;
    }
    return;
  }
  double beta;
  if (!cg_fused_step(v, st, rz_old, iter_old, alpha, pqv, beta)) return;
#pragma unroll
  for (int k = 0; k < FUSED_ITEMS; ++k) {
    const int64_t i = i0 + k * stride;
    if (i < n2) pn2[i] = make_double2(__fma_rn(beta, pk[k].x, zk[k].x), __fma_rn(beta, pk[k].y, zk[k].y));
  }
  for (int64_t i = i0 + FUSED_ITEMS * stride; i < n2; i += stride) {
    const double2 ri = r2[i], di = d2[i], pi = p2[i];
    pn2[i] = make_double2(__fma_rn(beta, pi.x, __dmul_rn(di.x, ri.x)), __fma_rn(beta, pi.y, __dmul_rn(di.y, ri.y)));
  }
}

// p_out = dinv r + beta p_in after a residual replacement of the fused form
__global__ void __launch_bounds__(256) cg_pfix_kernel(int ndof, const double* __restrict__ dinv,
                                                      const double* __restrict__ r,
                                                      const double* __restrict__ pin,
                                                      double* __restrict__ pout, const CgState* st,
                                                      BatchStrides bs) {
  {
    const int bd = blockIdx.y;
    dinv += bd * bs.dof;
    r += bd * bs.dof;
    pin += bd * bs.dof;
    pout += bd * bs.dof;
    st += bd;
  }
  if (st->done || !st->pfix) return;
  const double beta = st->beta;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride)
    pout[i] = __fma_rn(beta, pin[i], __dmul_rn(dinv[i], r[i]));
}

// f_bc = f with fixed DOFs zeroed; x = x0 (fixed zeroed) or 0; r = f_bc - K x0; p = z = dinv r.
__global__ void __launch_bounds__(256) cg_init_kernel(int ndof, const double* __restrict__ f,
                                                      const uint8_t* __restrict__ fixed_mask,
                                                      const double* __restrict__ dinv,
                                                      double* __restrict__ fbc,
                                                      double* __restrict__ x,
                                                      double* __restrict__ r,
                                                      double* __restrict__ p,
                                                      double* __restrict__ partial, CgState* st,
                                                      int warm, const double* __restrict__ Kx0,
                                                      BatchStrides bs) {
  __shared__ double sm[96];
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    f += bd * bs.dof;
    dinv += bd * bs.dof;
    fbc += bd * bs.dof;
    x += bd * bs.dof;
    r += bd * bs.dof;
    p += bd * bs.dof;
    Kx0 += bd * bs.dof;
    partial += bd * bs.partial;
    st += bd;
  }
  double v[3] = {0.0, 0.0, 0.0};  // f^T f, r^T z, r^T r
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride) {
    const bool fx = (fixed_mask[i / 6] >> (i % 6)) & 1;
    const double fi = fx ? 0.0 : f[i];
    fbc[i] = fi;
    double ri = fi;
    if (warm) {
      ri = fi - Kx0[i];
    } else {
      x[i] = 0.0;
    }
    r[i] = ri;
    const double zi = dinv[i] * ri;
    p[i] = zi;
    v[0] += fi * fi;
    v[1] += ri * zi;
    v[2] += ri * ri;
  }
  if (grid_sum<3>(v, partial, &st->ticket[2], sm) && threadIdx.x == 0) {
    st->ff = v[0];
    st->rz = v[1];
    st->rr = v[2];
    st->iter = 0;
    st->status = SSO_OK;
    st->done = (v[2] <= st->tol2 * v[0] || v[0] == 0.0) ? 1 : 0;
    st->tol2 = st->tol2 * v[0];  // host passes rtol^2 in tol2; becomes rtol^2 |f_bc|^2
    st->alpha = st->beta = 0.0;
    st->rr_ref = v[2];
  }
}

// zero fixed entries of x (warm start)
__global__ void zero_fixed_kernel(int ndof, const uint8_t* __restrict__ fixed_mask, double* x,
                                  BatchStrides bs) {
  x += blockIdx.y * bs.dof;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride)
    if ((fixed_mask[i / 6] >> (i % 6)) & 1) x[i] = 0.0;
}

__global__ void __launch_bounds__(256) residual_kernel(int ndof, const double* __restrict__ f,
                                                       const double* __restrict__ Kx,
                                                       double* __restrict__ partial,
                                                       CgState* st, BatchStrides bs) {
  __shared__ double sm[32];
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    f += bd * bs.dof;
    Kx += bd * bs.dof;
    partial += bd * bs.partial;
    st += bd;
  }
  double v[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride) {
    const double d = f[i] - Kx[i];
    v[0] += d * d;
  }
  if (grid_sum<1>(v, partial, &st->ticket[3], sm) && threadIdx.x == 0) st->red[0] = v[0];
}

// |f_bc - K x|^2 (local part) into red[0]; design from blockIdx.y.
__global__ void __launch_bounds__(256) cg_true_res_kernel(int ndof, const double* __restrict__ fbc,
                                                          const double* __restrict__ Kx,
                                                          double* __restrict__ partial, CgState* st,
                                                          BatchStrides bs) {
  __shared__ double sm[32];
  {
    const int bd = blockIdx.y;
    fbc += bd * bs.dof;
    Kx += bd * bs.dof;
    partial += bd * bs.partial;
    st += bd;
  }
  double v[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride) {
    const double d = fbc[i] - Kx[i];
    v[0] += d * d;
  }
  if (grid_sum<1>(v, partial, &st->ticket[3], sm) && threadIdx.x == 0) st->red[0] = v[0];
}

// Decide the residual replacement of every design (thread per design) from global values.
__global__ void cg_check_kernel(CgState* st, int mode, int B) {
  const int bd = blockIdx.x * blockDim.x + threadIdx.x;
  if (bd >= B) return;
  CgState* S = st + bd;
  // red[0] holds the global true |f_bc - K x|^2 of the current iterate
  const double tt = S->red[0];
  const bool drifted = tt > REPL_DRIFT * REPL_DRIFT * S->rr;
  if (mode == REPL_PERIODIC) {
    S->act = 0;
    if (!S->done && !S->floor && S->rr < REPL_FACTOR * S->rr_ref) {
      if (drifted) S->floor = 1;
      else S->act = (tt > REPL_CONT * REPL_CONT * S->rr) ? 2 : 1;
      if (S->act == 2) S->lz_frozen = 1;  // restart (beta = 0)
    }
  } else {
    S->act = 0;
    if (S->done && S->status == SSO_OK && !S->floor && tt > 4.0 * S->tol2 &&
        S->restarts < MAX_RESTARTS) {
      if (drifted && tt > 1e4 * S->tol2) {
        S->floor = 1;  // far from rtol because of the K x floor: restarting cannot help
      } else {
        S->act = 1;
        S->done = 0;
        S->restarts += 1;
        S->lz_frozen = 1;  // a restarted CG is a new Lanczos sequence: keep the first one
      }
    }
  }
}

// r = f_bc - K x for designs selected by cg_check; local r^T z, r^T r to red[]
// (partitioned) or straight into the state, with beta for the following p update
// (an iteration is p update -> SpMV -> x / r update, so r is replaced before p is formed).
__global__ void __launch_bounds__(256) cg_replace_kernel(int ndof, const double* __restrict__ fbc,
                                                         const double* __restrict__ Kx,
                                                         const double* __restrict__ dinv,
                                                         double* __restrict__ r, double* __restrict__ p,
                                                         double* __restrict__ partial, CgState* st,
                                                         int mode, BatchStrides bs) {
  __shared__ double sm[64];
  {
    const int bd = blockIdx.y;
    fbc += bd * bs.dof;
    Kx += bd * bs.dof;
    dinv += bd * bs.dof;
    r += bd * bs.dof;
    p += bd * bs.dof;
    partial += bd * bs.partial;
    st += bd;
  }
  if (!st->act) return;
  double v[2] = {0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride) {
    const double ri = fbc[i] - Kx[i];
    const double zi = dinv[i] * ri;
    r[i] = ri;
    v[0] += ri * zi;
    v[1] += ri * ri;
  }
  if (grid_sum<2>(v, partial, &st->ticket[1], sm) && threadIdx.x == 0) {
    st->rz = v[0];
    st->rr = v[1];
    st->rr_ref = v[1];
    // the next p update forms p = z + beta p: restart (final) -> beta = 0
    st->beta = (mode == REPL_FINAL || st->act == 2) ? 0.0 : v[0] / st->rz_prev;
    st->act = 0;
    st->pfix = 1;
  }
}

// buf[6k + c] = vec[6 idx[k] + c]  (halo send packing)
__global__ void pack_kernel(int count, const int32_t* __restrict__ idx, const double* __restrict__ vec,
                            double* __restrict__ buf) {
  const int64_t n = 6 * (int64_t)count;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = vec[6 * (int64_t)idx[i / 6] + (i % 6)];
}

// In-process allreduce over parts: red[v] = sum over parts in part order, written to all.
__global__ void allreduce_parts_kernel(CgState* const* sts, int n_parts, int nvals) {
  const int v = threadIdx.x;
  if (v >= nvals) return;
  double s = 0.0;
  for (int p = 0; p < n_parts; ++p) s += sts[p]->red[v];
  __syncwarp();
  for (int p = 0; p < n_parts; ++p) sts[p]->red[v] = s;
}

__global__ void gather_kernel(int n, const int32_t* __restrict__ idx, const double* __restrict__ src,
                              double* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

__global__ void scatter_kernel(int n, const int32_t* __restrict__ idx, const double* __restrict__ src,
                               double* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[idx[i]] = src[i];
}

__global__ void __launch_bounds__(256) dot_local_kernel(int n, const double* __restrict__ a,
                                                        const double* __restrict__ b,
                                                        double* __restrict__ partial,
                                                        CgState* st, BatchStrides bs) {
  __shared__ double sm[32];
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    a += bd * bs.dof;
    b += bd * bs.dof;
    partial += bd * bs.partial;
    st += bd;
  }
  double v[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) v[0] += a[i] * b[i];
  if (grid_sum<1>(v, partial, &st->ticket[3], sm) && threadIdx.x == 0) st->red[0] = v[0];
}

int vec_grid(int64_t n, int B = 1) {
  int64_t need = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)cg_grid() / B));
}

}  // namespace

void launch_cg_true_res(cudaStream_t s, int ndof, const double* fbc, const double* Kx, double* partial,
                        CgState* st, const BatchStrides& bs) {
  cg_true_res_kernel<<<dim3(vec_grid(ndof, bs.B), bs.B), 256, 0, s>>>(ndof, fbc, Kx, partial, st, bs);
  SSO_POST_LAUNCH("cg_true_res_kernel");
}

void launch_cg_check(cudaStream_t s, CgState* st, int mode, int B) {
  cg_check_kernel<<<(B + 127) / 128, 128, 0, s>>>(st, mode, B);
  SSO_POST_LAUNCH("cg_check_kernel");
}

void launch_cg_replace(cudaStream_t s, int ndof, const double* fbc, const double* Kx, const double* dinv,
                       double* r, double* p, double* partial, CgState* st, int mode, const BatchStrides& bs) {
  cg_replace_kernel<<<dim3(vec_grid(ndof, bs.B), bs.B), 256, 0, s>>>(ndof, fbc, Kx, dinv, r, p, partial, st,
                                                                     mode, bs);
  SSO_POST_LAUNCH("cg_replace_kernel");
}

namespace {
__global__ void lincomb_kernel(int64_t n, double a, const double* __restrict__ x, double b,
                               const double* __restrict__ y, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * x[i] + b * y[i];
}
}  // namespace


void launch_lincomb(cudaStream_t s, int64_t n, double a, const double* x, double b, const double* y, double* out) {
  if (n <= 0) return;
  lincomb_kernel<<<vec_grid(n), 256, 0, s>>>(n, a, x, b, y, out);
  SSO_POST_LAUNCH("lincomb_kernel");
}


void launch_pack(cudaStream_t s, int count, const int32_t* idx, const double* vec, double* buf) {
  if (count <= 0) return;
  pack_kernel<<<vec_grid(6 * (int64_t)count), 256, 0, s>>>(count, idx, vec, buf);
  SSO_POST_LAUNCH("pack_kernel");
}

void launch_allreduce_parts(cudaStream_t s, CgState* const* sts, int n_parts, int nvals) {
  allreduce_parts_kernel<<<1, 32, 0, s>>>(sts, n_parts, nvals);
  SSO_POST_LAUNCH("allreduce_parts_kernel");
}

void launch_gather(cudaStream_t s, int n, const int32_t* idx, const double* src, double* dst) {
  if (n <= 0) return;
  gather_kernel<<<vec_grid(n), 256, 0, s>>>(n, idx, src, dst);
  SSO_POST_LAUNCH("gather_kernel");
}

void launch_scatter(cudaStream_t s, int n, const int32_t* idx, const double* src, double* dst) {
  if (n <= 0) return;
  scatter_kernel<<<vec_grid(n), 256, 0, s>>>(n, idx, src, dst);
  SSO_POST_LAUNCH("scatter_kernel");
}

void launch_dot_local(cudaStream_t s, int n, const double* a, const double* b, double* partial,
                      CgState* st, const BatchStrides& bs) {
  dot_local_kernel<<<dim3(vec_grid(n, bs.B), bs.B), 256, 0, s>>>(n, a, b, partial, st, bs);
  SSO_POST_LAUNCH("dot_local_kernel");
}

int cg_grid() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms * 4;  // 4 CTAs x 256 threads per SM, every grid a multiple of the SM count
}

void launch_cg_init(cudaStream_t s, int ndof, const double* f, const uint8_t* fixed_mask,
                    const double* dinv, double* fbc, double* x, double* r, double* p,
                    double* partial, CgState* st, int warm, const double* Kx0,
                    const BatchStrides& bs) {
  cg_init_kernel<<<dim3(vec_grid(ndof, bs.B), bs.B), 256, 0, s>>>(ndof, f, fixed_mask, dinv, fbc, x, r, p,
                                                                partial, st, warm, Kx0, bs);
  SSO_POST_LAUNCH("cg_init_kernel");
}

void launch_zero_fixed(cudaStream_t s, int ndof, const uint8_t* fixed_mask, double* x,
                       const BatchStrides& bs) {
  zero_fixed_kernel<<<dim3(vec_grid(ndof, bs.B), bs.B), 256, 0, s>>>(ndof, fixed_mask, x, bs);
  SSO_POST_LAUNCH("zero_fixed_kernel");
}

struct SpmvVariant {
  int stages, slot_deg, minb;
  void (*dot)(int, int, const int64_t*, const int32_t*, const double*, const double*, double*,
              double*, CgState*, BatchStrides);
  void (*plain)(int, int, const int64_t*, const int32_t*, const double*, const double*, double*,
                double*, CgState*, BatchStrides);
};
#define SPMV_VARIANT(S, D, M) \
  { S, D, M, spmv_tma_kernel<true, S, D, M>, spmv_tma_kernel<false, S, D, M> }
static const SpmvVariant kSpmvVariants[] = {
    SPMV_VARIANT(4, 10, 2), SPMV_VARIANT(3, 10, 3), SPMV_VARIANT(2, 9, 4), SPMV_VARIANT(3, 9, 3),
    SPMV_VARIANT(2, 10, 4)};


static const SpmvVariant& spmv_variant() {
  static int v = -1;
  static uint64_t attr_mask = 0;
  if (v < 0) {
    const char* e = getenv("SSO_SPMV_VARIANT");
    v = e ? atoi(e) : 2;  // default: 2-slot ring, 4 CTAs per SM (measured best at C3b)
    const int nv = (int)(sizeof(kSpmvVariants) / sizeof(kSpmvVariants[0]));
    if (v < 0 || v >= nv) v = 0;
  }
  const SpmvVariant& V = kSpmvVariants[v];
  if (first_on_device(attr_mask)) {
    const int smem = SPMV_WARPS * V.stages * 36 * V.slot_deg * 8;
    cudaFuncSetAttribute(V.dot, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(V.plain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  return V;
}

static void spmv_config(int n_nodes, int B, int* grid, int* npw, int* smem) {
  const SpmvVariant& V = spmv_variant();
  const int ctas = std::max(1, V.minb * (cg_grid() / 4) / B);  // persistent: minb CTAs per SM in total
  const int64_t warps = (int64_t)ctas * SPMV_WARPS;
  int per = (int)((n_nodes + warps - 1) / warps);
  if (per < 1) per = 1;
  *npw = per;
  *grid = (int)std::max<int64_t>(1, (((int64_t)n_nodes + per - 1) / per + SPMV_WARPS - 1) / SPMV_WARPS);
  *smem = SPMV_WARPS * V.stages * 36 * V.slot_deg * 8;
}

void launch_spmv_dot(cudaStream_t s, int n_nodes, const int64_t* node_ptr, const int32_t* node_col,
                     const double* vals, const double* p, double* q, double* partial, CgState* st,
                     const BatchStrides& bs) {
  int grid, npw, smem;
  spmv_config(n_nodes, bs.B, &grid, &npw, &smem);
  spmv_variant().dot<<<dim3(grid, bs.B), SPMV_WARPS * 32, smem, s>>>(n_nodes, npw, node_ptr, node_col, vals,
                                                                     p, q, partial, st, bs);
  SSO_POST_LAUNCH("spmv_dot_kernel");
}

// pull SpMV (storage 3).  Variants (chunk nodes, buffers, CTAs per SM, consumer warps):
// 0 (12, 2, 3, 4) single designs, 1 (8, 2, 4, 4) batches, 2 (16, 2, 2, 8), 3 (8, 3, 3, 4).
// Measured at C3b: 67.0, 68.4, 69.9, 71.6 us; also tried (live us): (4, 2, 8, 2) 75.9,
// (16, 2, 2, 4) 72.3, (12, 2, 3, 6) 93 (spills), (10, 2, 3, 5) 71.7, (12, 3, 2, 4) 76.0,
// (12, 2, 3, 3) 70.5, (9, 2, 4, 3) 67.5, (6, 2, 5, 3) 69.1, (15, 2, 2, 5) 69.6.  Finer chunks
// pay the producer per chunk, larger ones limit the
// CTAs per SM (shared memory) or spill.
struct PullVariant {
  int smem;
  int minb;
  int threads;
  int chunk;  // nodes per CTA chunk
  void (*dot)(const CUtensorMap, int, int, int, int, const int32_t*, const int32_t*, const int2*, const double*,
              const double*, double*, double*, CgState*, BatchStrides, const PullPart*);
  void (*plain)(const CUtensorMap, int, int, int, int, const int32_t*, const int32_t*, const int2*, const double*,
                const double*, double*, double*, CgState*, BatchStrides, const PullPart*);
};
#define PULL_CTA_VARIANT(C, NB, M, W)                                                                 \
  {                                                                                                   \
    (NB * PullChunkSmem<C, W>::BUF + W * PullChunkSmem<C, W>::RED) * 8, M, 32 * (W + 1), C,           \
        spmv_pull_cta_kernel<true, C, NB, M, W>, spmv_pull_cta_kernel<false, C, NB, M, W>             \
  }
static const PullVariant kPullVariants[] = {PULL_CTA_VARIANT(12, 2, 3, 4), PULL_CTA_VARIANT(8, 2, 4, 4),
                                            PULL_CTA_VARIANT(16, 2, 2, 8), PULL_CTA_VARIANT(8, 3, 3, 4)};
// Variant per launch: SSO_PULL_VARIANT if set, else 0 for single designs and 1 (8-node
// chunks, more CTAs per design) for batches (C5: 220 vs 206 designs/s).
static const PullVariant& pull_variant(int B, int* smem) {
  static int env_v = -2;
  static uint64_t attr_mask[sizeof(kPullVariants) / sizeof(kPullVariants[0])] = {};
  const int nv = (int)(sizeof(kPullVariants) / sizeof(kPullVariants[0]));
  if (env_v == -2) {
    const char* e = getenv("SSO_PULL_VARIANT");
    env_v = e ? atoi(e) : -1;
    if (env_v >= nv) env_v = -1;
  }
  const int v = env_v >= 0 ? env_v : (B > 1 ? 1 : 0);
  if (first_on_device(attr_mask[v])) {
    cudaFuncSetAttribute(kPullVariants[v].dot, cudaFuncAttributeMaxDynamicSharedMemorySize, kPullVariants[v].smem);
    cudaFuncSetAttribute(kPullVariants[v].plain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kPullVariants[v].smem);
  }
  *smem = kPullVariants[v].smem;
  return kPullVariants[v];
}

void build_pull_desc(const UpperPattern& U, std::vector<int32_t>& d) {
  const int64_t nn = (int64_t)U.uptr.size() - 1;
  d.assign((size_t)(PULL_DESC * nn), 0);
  for (int64_t m = 0; m < nn; ++m) {
    int32_t* o = d.data() + PULL_DESC * m;
    const int64_t b0 = U.uptr[m], l0 = U.lptr[m];
    const int udeg = (int)(U.uptr[m + 1] - b0), ldeg = (int)(U.lptr[m + 1] - l0);
    const bool fits = udeg <= PULL_MAX_UDEG && ldeg <= 4;
    o[0] = (int32_t)b0;
    o[1] = (std::min(udeg, 255)) | (std::min(ldeg, 255) << 8) | ((fits ? 1 : 0) << 16);
    if (!fits) {
      o[2] = (int32_t)l0;
      continue;
    }
    for (int k = 0; k < udeg; ++k) o[2 + k] = U.ucol[b0 + k];
    for (int j = 0; j < ldeg; ++j) {
      o[2 + udeg + 2 * j] = U.lpull[2 * (l0 + j)];
      o[3 + udeg + 2 * j] = U.lpull[2 * (l0 + j) + 1];
    }
  }
}

int make_pull_tmap(const double* vals, int64_t rows, CUtensorMap* out) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess || !fn)
      return 1;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  // [rows][PULL_BLOCK] fp64 view of the values; a box is one record, gather4 fetches four
  cuuint64_t dims[2] = {PULL_BLOCK, (cuuint64_t)rows};
  cuuint64_t strides[1] = {8 * PULL_BLOCK};
  cuuint32_t box[2] = {PULL_BLOCK, 1};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(vals), dims, strides,
                            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 2;
}

void launch_spmv_pull(cudaStream_t s, const CUtensorMap* tmap, int n_nodes, int rows_per_design,
                      const int32_t* pdesc, const int32_t* ucol, const int32_t* lpull, const double* vals,
                      const double* x, double* y, double* partial, CgState* st, const BatchStrides& bs, int node0,
                      int red_add, int share) {
  if (n_nodes <= node0) return;
  int smem;
  const PullVariant& V = pull_variant(bs.B, &smem);
  // persistent: minb CTAs per SM in total, divided among `share` concurrently running launches
  const int ctas = std::max(1, V.minb * (cg_grid() / 4) / (bs.B * std::max(share, 1)));
  const int chunk = V.chunk;
  const int units = (n_nodes - node0 + chunk - 1) / chunk;
  const int grid = std::max(1, std::min(ctas, units));
  const int2* lp = reinterpret_cast<const int2*>(lpull);
  if (st)
    V.dot<<<dim3(grid, bs.B), V.threads, smem, s>>>(*tmap, n_nodes, node0, red_add, rows_per_design, pdesc, ucol, lp,
                                                         vals, x, y, partial, st, bs, nullptr);
  else
    V.plain<<<dim3(grid, bs.B), V.threads, smem, s>>>(*tmap, n_nodes, node0, red_add, rows_per_design, pdesc, ucol,
                                                           lp, vals, x, y, nullptr, nullptr, bs, nullptr);
  SSO_POST_LAUNCH(st ? "spmv_pull_dot_kernel" : "spmv_pull_kernel");
}

void launch_spmv_pull_multi(cudaStream_t s, const PullPart* mp, int n_parts, int max_nodes) {
  if (n_parts <= 0 || max_nodes <= 0) return;
  int smem;
  const PullVariant& V = pull_variant(1, &smem);  // the single-design variant: parts are large
  const int ctas = std::max(1, V.minb * (cg_grid() / 4) / n_parts);  // the parts side by side
  const int units = (max_nodes + V.chunk - 1) / V.chunk;
  const int grid = std::max(1, std::min(ctas, units));
  // the per-launch tensor map parameter is unused (each part brings its own)
  CUtensorMap dummy;
  std::memset(&dummy, 0, sizeof dummy);
  V.dot<<<dim3(grid, n_parts), V.threads, smem, s>>>(dummy, max_nodes, 0, 0, 0, nullptr, nullptr, nullptr, nullptr,
                                                          nullptr, nullptr, nullptr, nullptr, BatchStrides(), mp);
  SSO_POST_LAUNCH("spmv_pull_dot_kernel (parts)");
}

void launch_spmv(cudaStream_t s, int n_nodes, const int64_t* node_ptr, const int32_t* node_col,
                 const double* vals, const double* x, double* y, const BatchStrides& bs) {
  int grid, npw, smem;
  spmv_config(n_nodes, bs.B, &grid, &npw, &smem);
  spmv_variant().plain<<<dim3(grid, bs.B), SPMV_WARPS * 32, smem, s>>>(n_nodes, npw, node_ptr, node_col,
                                                                       vals, x, y, nullptr, nullptr, bs);
  SSO_POST_LAUNCH("spmv_kernel");
}



void launch_cg_update(cudaStream_t s, int ndof, const double* dinv, double* x, double* r,
                      const double* p, const double* q, double* partial, CgState* st,
                      const BatchStrides& bs) {
  cg_update_kernel<<<dim3(vec_grid(ndof, bs.B), bs.B), 256, 0, s>>>(ndof, dinv, x, r, p, q, partial, st, bs);
  SSO_POST_LAUNCH("cg_update_kernel");
}

int cg_fused_grid() {
  static int g = -1;
  if (g < 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cg_update_fused_kernel, 256, 0) != cudaSuccess) occ = 0;
    cg_grid();
    g = std::min(occ, 2) * g_sms;
  }
  return g;
}

void launch_cg_update_fused(cudaStream_t s, int ndof, const double* dinv, double* x, double* r,
                            const double* p, const double* q, double* pn, double* partial, CgState* st,
                            const BatchStrides& bs) {
  // every CTA of every design co-resident (bs.B <= cg_fused_grid(), checked at create)
  const int64_t need = ((int64_t)ndof / 2 + 255) / 256;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, cg_fused_grid() / bs.B));
  const cudaError_t e = launch_cooperative(cg_update_fused_kernel, dim3(grid, bs.B), dim3(256), s, ndof, dinv, x, r,
                                           p, q, pn, partial, st, bs);
  SSO_POST_LAUNCH_RC("cg_update_fused_kernel", e);
}

void launch_cg_pfix(cudaStream_t s, int ndof, const double* dinv, const double* r, const double* pin,
                    double* pout, const CgState* st, const BatchStrides& bs) {
  cg_pfix_kernel<<<dim3(vec_grid(ndof, bs.B), bs.B), 256, 0, s>>>(ndof, dinv, r, pin, pout, st, bs);
  SSO_POST_LAUNCH("cg_pfix_kernel");
}

void launch_cg_pupdate(cudaStream_t s, int ndof, const double* dinv, const double* r, double* p,
                       CgState* st, const BatchStrides& bs) {
  cg_pupdate_kernel<<<dim3(vec_grid(ndof, bs.B), bs.B), 256, 0, s>>>(ndof, dinv, r, p, st, bs);
  SSO_POST_LAUNCH("cg_pupdate_kernel");
}

void launch_residual_norm(cudaStream_t s, int ndof, const double* f, const double* Kx,
                          double* partial, CgState* st, const BatchStrides& bs) {
  residual_kernel<<<dim3(vec_grid(ndof, bs.B), bs.B), 256, 0, s>>>(ndof, f, Kx, partial, st, bs);
  SSO_POST_LAUNCH("residual_kernel");
}

}  // namespace sso
