// A3 SpMV, "sweep" form of the upper-block storage (storage 3 records; sm_100a).
//
// y = K x with K symmetric and only the upper node blocks (n, m >= n) stored (DESIGN.md §5:
// 38-double records of nine 2x2 sub-blocks).  The pull kernel (pcg.cu) reads every stored
// block twice -- once by its row node n (K_nm x_m) and, gathered from L2, once by its column
// node m (K_nm^T x_n).  Here every block is read ONCE and used twice:
//
//   * the node range of a design is split into G contiguous ranges, one persistent CTA each
//     (cooperative launch, one or two CTAs per SM); a CTA sweeps its range in chunks of C
//     consecutive nodes whose upper runs are contiguous in memory (one bulk copy per chunk,
//     a producer warp, W chunk buffers, W consumer warps: warp w takes chunks w, w + W, ...);
//   * consumer lane (block k, column pair B; two nodes per warp pass) loads the three 2x2 sub-blocks (A, B), A = 0..2,
//     of its block once and forms both the row-node partials K[., 2B..2B+1] x_m[2B..2B+1] and
//     the column-node outputs (K^T x_n)[2B..2B+1] of the block (complete in the lane);
//   * the K^T x_n contribution to node m > n is stored in a shared-memory RING of per-node
//     slots (slot s = position of n in m's ascending lower-neighbour list: every (m, s) has
//     exactly one writer, no atomics); m's row is finalised when its own chunk is done and
//     every earlier chunk of the range has stored its contributions (an in-order
//     "products done" counter): q_m = (own row sum) + sum over slots in ascending source
//     order -- deterministic;
//   * the mesh bandwidth bw (max m - n over stored blocks) bounds how far ahead a
//     contribution lands, so the ring holds bw + (2W + 1) C nodes (C3b: 410 + 104); the
//     contributions to the next range's first bw nodes are handed over through a global
//     carry buffer at the end of the sweep (per-range completion counters, acquire /
//     release), and added by the next CTA to its first bw rows after its own sweep.
//
// Applies when every owned node has at most 5 upper and 4 lower neighbours (grid shells)
// and the ring fits in shared memory (bw up to ~550 nodes at C = 8, W = 6); otherwise the
// pull kernel runs.  Bytes per launch: the stored records once (no L2 gathers of pulled
// records), 64 B of descriptor per node, x gathers, q written.
#include <cuda.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "cg_common.cuh"
#include "sso_internal.h"
#include "tma.cuh"

namespace sso {

namespace {

constexpr int SW_C = 8;   // nodes per chunk
constexpr int SW_W = 12;  // consumer warps = chunk buffers
constexpr int SW_MAXU = 5, SW_MAXL = 4;

constexpr int SW_XR = 4;     // x runs per chunk
constexpr int SW_XMAX = 48;  // x rows per chunk (6 doubles each)

struct SweepSmem {
  static constexpr int BUF = SW_C * SW_MAXU * PULL_BLOCK;  // doubles per chunk buffer: upper runs
  static constexpr int XBUF = SW_XMAX * 6;                 // doubles per chunk buffer: x rows
  static constexpr int DESC = SW_C * SWEEP_DESC;           // ints per chunk descriptor copy
  static constexpr int OWN = SW_C * 6;                     // doubles per warp: own row sums of a chunk
  static size_t bytes() { return (size_t)SW_W * (BUF + XBUF + OWN) * 8 + (size_t)SW_W * DESC * 4; }
};

__device__ __forceinline__ unsigned ld_acquire_cta(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(unsigned* p, unsigned v) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool DOT>
__global__ void __launch_bounds__(32 * SW_W, 1) spmv_sweep_kernel(
    int n_own, int L, int bw, int R, const int32_t* __restrict__ sdesc, const int64_t* __restrict__ uptr,
    const int2* __restrict__ xrun, const double* __restrict__ vals,
    const double* __restrict__ p, double* __restrict__ q, double* __restrict__ partial, CgState* st,
    double* __restrict__ carry, unsigned* __restrict__ flags, int red_add, BatchStrides bs, int dbg) {
  using S = SweepSmem;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[SW_W];
  __shared__ unsigned done_upto;  // chunks [0, done_upto) have stored their ring contributions
  __shared__ unsigned s_epoch;
  __shared__ double sm[32];
  const int bd = blockIdx.y, G = gridDim.x, r = blockIdx.x;
  vals += bd * bs.nnz;
  p += bd * bs.dof;
  q += bd * bs.dof;
  if (DOT) {
    partial += bd * bs.partial;
    st += bd;
    if (st->done) return;
  }
  double* __restrict__ gst = carry + (int64_t)bd * n_own * 24;  // [n_own][4 slots][6]
  flags += bd * G;
  const int a = r * L, b = min(n_own, a + L);
  const int nchunk = (b - a + SW_C - 1) / SW_C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* buf0 = reinterpret_cast<double*>(smem_raw);
  double* xbuf0 = buf0 + (size_t)SW_W * S::BUF;
  double* own0 = xbuf0 + (size_t)SW_W * S::XBUF;
  int32_t* desc0 = reinterpret_cast<int32_t*>(own0 + (size_t)SW_W * S::OWN);
  if (tid == 0) {
    for (int w = 0; w < SW_W; ++w) {
      mbar_init(&full_bar[w], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    done_upto = 0;
    s_epoch = *reinterpret_cast<volatile unsigned*>(flags + r);
  }
  __syncthreads();
  double pq = 0.0;
  {
    // Every warp is its own producer and consumer: warp w takes chunks w, w + W, ... into its
    // buffer.  Per chunk, lane 0 issues bulk copies of the descriptors, the upper runs and the
    // x rows the chunk reads (host-listed runs of consecutive nodes) on the buffer's barrier;
    // the chunk's record range and x runs ("meta") are loaded one chunk ahead, so issuing never
    // waits on a global load, and the copies of chunk k + W are issued as soon as chunk k is
    // done (W chunks in flight per CTA, issued from W warps in parallel).
    const int w = warp;
    const uint64_t pol = evict_first_policy();
    // meta of chunk k: lane 0 / 1 the record range ends, lanes 2 .. 2 + SW_XR - 1 the x runs
    auto load_meta = [&](int k) -> int2 {
      int2 v = make_int2(0, 0);
      if (k < nchunk) {
        const int first = a + k * SW_C, last = min(b, first + SW_C);
        if (lane == 0) v.x = (int)uptr[first];
        else if (lane == 1) v.x = (int)uptr[last];
        else if (lane < 2 + SW_XR) v = xrun[SW_XR * (int64_t)(first / SW_C) + (lane - 2)];
      }
      return v;
    };
    auto issue = [&](int k, int2 mv) {
      const int bf = __shfl_sync(FULL, mv.x, 0), be = __shfl_sync(FULL, mv.x, 1);
      int2 run[SW_XR];
      int xrows = 0;
#pragma unroll
      for (int j = 0; j < SW_XR; ++j) {
        run[j].x = __shfl_sync(FULL, mv.x, 2 + j);
        run[j].y = __shfl_sync(FULL, mv.y, 2 + j);
        xrows += run[j].y;
      }
      if (lane == 0 && k < nchunk) {
        const int first = a + k * SW_C, nc = min(SW_C, b - first);
        // generic reads of this buffer (previous chunk) precede the async writes below
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const unsigned dbytes = (unsigned)(4 * SWEEP_DESC * nc), rbytes = (unsigned)(8 * PULL_BLOCK * (be - bf));
        mbar_arrive_expect_tx(&full_bar[w], dbytes + rbytes + ((dbg & 2) ? 0u : (unsigned)(48 * xrows)));
        bulk_g2s(desc0 + (size_t)w * S::DESC, sdesc + SWEEP_DESC * (int64_t)first, dbytes, &full_bar[w], pol);
        bulk_g2s(buf0 + (size_t)w * S::BUF, vals + PULL_BLOCK * (int64_t)bf, rbytes, &full_bar[w], pol);
        double* xd = xbuf0 + (size_t)w * S::XBUF;
#pragma unroll
        for (int j = 0; j < SW_XR; ++j)
          if (run[j].y > 0 && !(dbg & 2)) {
            bulk_g2s_plain(xd, p + 6 * (int64_t)run[j].x, (unsigned)(48 * run[j].y), &full_bar[w]);
            xd += 6 * run[j].y;
          }
      }
      __syncwarp();
    };
    issue(w, load_meta(w));
    int2 meta_next = load_meta(w + SW_W);
    const double* buf = buf0 + (size_t)w * S::BUF;
    const double* xb = xbuf0 + (size_t)w * S::XBUF;
    double* own = own0 + (size_t)w * S::OWN;
    const int32_t* D = desc0 + (size_t)w * S::DESC;
    // lane -> (node of the pass = lane / 16, block k, column pair B); lane 15 of each half idle.
    // A pass covers two nodes; every operand is in shared memory (no global load on the chain).
    const int ns = lane >> 4, u = lane & 15, kb = u / 3, Bc = u - 3 * (u / 3);
    int offs[3];
#pragma unroll
    for (int A = 0; A < 3; ++A) offs[A] = pull_sub_off(3 * Bc + A);
    constexpr int NP = SW_C / 2;              // passes per chunk
    constexpr int NF = (6 * SW_C + 31) / 32;  // finalise iterations per chunk
    for (int k = w, it = 0; k < nchunk; k += SW_W, ++it) {
      const int first = a + k * SW_C, nc = min(SW_C, b - first);
      {  // start pulling chunk k + W's upper runs into L2 (its shared-memory copy follows chunk k)
        const int pf0 = __shfl_sync(FULL, meta_next.x, 0), pf1 = __shfl_sync(FULL, meta_next.x, 1);
        if (lane == 0 && k + SW_W < nchunk && !(dbg & 8))
          bulk_prefetch_l2(vals + PULL_BLOCK * (int64_t)pf0, (unsigned)(8 * PULL_BLOCK * (pf1 - pf0)));
      }
      mbar_wait(&full_bar[w], (unsigned)(it & 1));
      const int b_first = D[0];
#pragma unroll
      for (int ps = 0; ps < ((dbg & 4) ? 0 : NP); ++ps) {
        const int i = 2 * ps + ns;
        const int* Di = D + SWEEP_DESC * (i < nc ? i : 0);
        const bool act = u < 15 && i < nc && kb < (Di[1] & 255);
        double o[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (act) {
          const unsigned xp = (unsigned)Di[15];
          const double* xm = xb + 6 * ((xp >> (6 * kb)) & 63) + 2 * Bc;
          const double* xn = xb + 6 * (xp & 63);
          const double2 xmv = *reinterpret_cast<const double2*>(xm);
          const double2 xn0 = *reinterpret_cast<const double2*>(xn);
          const double2 xn1 = *reinterpret_cast<const double2*>(xn + 2);
          const double2 xn2 = *reinterpret_cast<const double2*>(xn + 4);
          const double* rec = buf + PULL_BLOCK * (Di[0] - b_first + kb);
          double t0 = 0.0, t1 = 0.0;
#pragma unroll
          for (int A = 0; A < 3; ++A) {
            // sub-block (A, B): K[2A][2B], K[2A+1][2B] | K[2A][2B+1], K[2A+1][2B+1]
            const double2 c0 = *reinterpret_cast<const double2*>(rec + offs[A]);
            const double2 c1 = *reinterpret_cast<const double2*>(rec + offs[A] + 2);
            const double2 xa = A == 0 ? xn0 : (A == 1 ? xn1 : xn2);
            o[2 * A] = fma(c0.x, xmv.x, c1.x * xmv.y);
            o[2 * A + 1] = fma(c0.y, xmv.x, c1.y * xmv.y);
            t0 = fma(c0.x, xa.x, fma(c0.y, xa.y, t0));
            t1 = fma(c1.x, xa.x, fma(c1.y, xa.y, t1));
          }
          if (kb >= 1) {
            const int slot = Di[6 + kb];
            if (slot >= 0) {
              const int m = Di[2 + kb];
              __stcg(reinterpret_cast<double2*>(gst + (size_t)m * 24 + 6 * slot + 2 * Bc), make_double2(t0, t1));
            }
          }
        }
        // own row sums of the pass's two nodes: butterfly over the 16 lanes of each half
#pragma unroll
        for (int off = 8; off > 0; off >>= 1)
#pragma unroll
          for (int rr = 0; rr < 6; ++rr) o[rr] += __shfl_xor_sync(FULL, o[rr], off);
        if (u < 6) {
          const double v = u == 0 ? o[0] : u == 1 ? o[1] : u == 2 ? o[2] : u == 3 ? o[3] : u == 4 ? o[4] : o[5];
          own[6 * (2 * ps + ns) + u] = v;
        }
      }
      // publish this chunk's ring contributions in chunk order
      __syncwarp();
      if (lane == 0) {
        // bounded: a broken chain reports SSO_E_CUDA instead of hanging the device
        int spin = 0;
        while (!(dbg & 1) && ld_acquire_cta(&done_upto) != (unsigned)k && ++spin < (1 << 22)) __nanosleep(32);
        if (spin >= (1 << 22) && DOT) {
          st->status = SSO_E_CUDA;
          st->done = 1;
        }
        st_release_cta(&done_upto, (unsigned)(k + 1));
      }
      __syncwarp();
      // every earlier chunk of the range has stored its contributions: finalise the chunk's rows
#pragma unroll
      for (int t = 0; t < NF; ++t) {
        const int idx = 32 * t + lane;
        if (idx < 6 * nc) {
          const int i = idx / 6, row = idx - 6 * (idx / 6);
          const int* Di = D + SWEEP_DESC * i;
          const int n = first + i;
          const int ldeg = (Di[1] >> 8) & 255;
          double y = own[6 * i + row];
          const double* rg = gst + (size_t)n * 24 + row;
          for (int s2 = 0; s2 < ldeg; ++s2)
            if (Di[11 + s2] >= a) y += __ldcg(rg + 6 * s2);
          q[6 * (int64_t)n + row] = y;
          if (DOT) pq = fma(xb[6 * (Di[15] & 63) + row], y, pq);
        }
      }
      __syncwarp();
      // this buffer is free: the copies of chunk k + W, then the meta of chunk k + 2W
      issue(k + SW_W, meta_next);
      meta_next = load_meta(k + 2 * SW_W);
    }
  }
  __syncthreads();
  // hand the contributions to the next range's first bw nodes over; take ours from the previous
  const unsigned epoch = s_epoch;
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release_gpu(flags + r, epoch + 1);
  if (r > 0) {
    __shared__ int s_ok;
    if (tid == 0) {
      int ok = 0;
      for (int spin = 0; spin < (1 << 24); ++spin) {
        if ((int)(ld_acquire_gpu(flags + r - 1) - (epoch + 1)) >= 0) {
          ok = 1;
          break;
        }
        __nanosleep(64);
      }
      s_ok = ok;
    }
    __syncthreads();
    if (s_ok) {
      const int m_end = min(b, a + bw);
      for (int idx = tid; idx < 6 * (m_end - a); idx += blockDim.x) {
        const int mm = idx / 6, row = idx - 6 * mm;
        const int n = a + mm;
        const int* Dn = sdesc + SWEEP_DESC * (int64_t)n;
        const int ldeg = (Dn[1] >> 8) & 255;
        double d = 0.0;
        for (int s = 0; s < ldeg; ++s)
          if (Dn[11 + s] < a) d += __ldcg(gst + (size_t)n * 24 + 6 * s + row);
        if (ldeg > 0 && Dn[11] < a) {
          q[6 * (int64_t)n + row] += d;
          if (DOT) pq = fma(p[6 * (int64_t)n + row], d, pq);
        }
      }
    } else if (DOT && tid == 0) {
      st->status = SSO_E_CUDA;  // the previous range never finished: report instead of hanging
      st->done = 1;
    }
  }
  if (DOT) {
    double v[1] = {pq};
    if (st->defer_alpha) {
      block_sum<1>(v, sm);
      if (tid == 0) {
        partial[PQ_OFF + blockIdx.x] = v[0];
        if (blockIdx.x == 0) st->npq = (int)gridDim.x;
      }
    } else if (grid_sum<1>(v, partial, &st->ticket[0], sm) && tid == 0) {
      if (st->dist) {
        st->red[0] = (red_add ? st->red[0] : 0.0) + v[0];
        return;
      }
      st->pq = v[0];
      if (!(v[0] > 0.0)) {
        st->status = SSO_E_NOT_SPD;
        st->done = 1;
      } else {
        st->alpha = st->rz / v[0];
      }
    }
  }
}

}  // namespace

// Host plan (see sso_internal.h SweepPlan): per-node descriptors, the bandwidth, ranges.
bool build_sweep_plan(const UpperPattern& U, int32_t n_own, int sms, int B, SweepPlan& plan) {
  plan = SweepPlan();
  const int64_t nn = (int64_t)U.uptr.size() - 1;
  if (n_own <= 0 || nn < n_own) return false;
  std::vector<int32_t>& d = plan.desc;
  d.assign((size_t)SWEEP_DESC * n_own, 0);
  int bw = 1;
  for (int32_t n = 0; n < n_own; ++n) {
    const int64_t b0 = U.uptr[n], l0 = U.lptr[n];
    const int udeg = (int)(U.uptr[n + 1] - b0), ldeg = (int)(U.lptr[n + 1] - l0);
    if (udeg > SW_MAXU || ldeg > SW_MAXL || udeg < 1 || U.ucol[b0] != n) return false;
    int32_t* o = d.data() + SWEEP_DESC * (int64_t)n;
    o[0] = (int32_t)b0;
    o[1] = udeg | (ldeg << 8);
    for (int k = 0; k < udeg; ++k) o[2 + k] = U.ucol[b0 + k];
    for (int k = 1; k < udeg; ++k) {
      const int32_t m = U.ucol[b0 + k];
      int slot = -1;
      if (m < n_own) {
        bw = std::max(bw, m - n);
        for (int64_t j = U.lptr[m]; j < U.lptr[m + 1]; ++j)
          if (U.lpull[2 * j] == n) slot = (int)(j - U.lptr[m]);
        if (slot < 0) return false;
      }
      o[6 + k] = slot;
    }
    for (int s = 0; s < ldeg; ++s) o[11 + s] = U.lpull[2 * (l0 + s)];
  }
  // x rows of every chunk (global chunks of SW_C nodes: ranges are chunk-aligned) as at most
  // SW_XR runs of consecutive nodes, <= SW_XMAX rows; each node's descriptor word 15 packs the
  // positions (6 bits each) of its upper neighbours' rows in the chunk's x buffer
  const int64_t nch = (n_own + SW_C - 1) / SW_C;
  plan.xrun.assign((size_t)(2 * SW_XR) * nch, 0);
  std::vector<int32_t> need;
  for (int64_t c = 0; c < nch; ++c) {
    const int32_t n0 = (int32_t)(c * SW_C), n1 = (int32_t)std::min<int64_t>(n_own, (c + 1) * SW_C);
    need.clear();
    for (int32_t n = n0; n < n1; ++n)
      for (int64_t j = U.uptr[n]; j < U.uptr[n + 1]; ++j) need.push_back(U.ucol[j]);
    std::sort(need.begin(), need.end());
    need.erase(std::unique(need.begin(), need.end()), need.end());
    if ((int)need.size() > SW_XMAX) return false;
    int nr = 0;
    for (size_t j = 0; j < need.size(); ++j) {
      if (j == 0 || need[j] != need[j - 1] + 1) {
        if (nr == SW_XR) return false;
        plan.xrun[2 * (SW_XR * c + nr)] = need[j];
        ++nr;
      }
      plan.xrun[2 * (SW_XR * c + nr - 1) + 1] += 1;
    }
    for (int32_t n = n0; n < n1; ++n) {
      int32_t* o = d.data() + SWEEP_DESC * (int64_t)n;
      const int udeg = o[1] & 255;
      uint32_t pos = 0;
      for (int k = 0; k < udeg; ++k) {
        const int at = (int)(std::lower_bound(need.begin(), need.end(), o[2 + k]) - need.begin());
        pos |= (uint32_t)at << (6 * k);
      }
      o[15] = (int32_t)pos;
    }
  }
  plan.bw = bw;
  plan.R = 0;
  plan.smem = (int)SweepSmem::bytes();
  if (plan.smem > 227 * 1024 - 1024) return false;  // static shared memory of the kernel on top
  // ranges: G per design, each at least bw nodes long (contributions reach the next range only)
  // and a multiple of the chunk; two CTAs per SM when the shared memory allows
  const int per_sm = plan.smem <= 113 * 1024 ? 2 : 1;
  int G = std::max(1, sms * per_sm / std::max(B, 1));
  G = std::min<int64_t>(G, std::max<int64_t>(1, n_own / std::max(bw, SW_C)));
  int L = (n_own + G - 1) / G;
  L = (L + SW_C - 1) / SW_C * SW_C;
  if (G > 1 && L < bw) return false;
  G = (n_own + L - 1) / L;
  plan.G = G;
  plan.L = L;
  return true;
}

int sweep_config_ok(const SweepPlan& plan, int B) {
  // the kernel's dynamic shared memory limit is raised to what this plan needs (per device; a
  // failed attribute call must not leave an error behind for a later launch check)
  static int set_bytes[64] = {0};
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) d = 0;
  if (set_bytes[d] < plan.smem) {
    if (cudaFuncSetAttribute(spmv_sweep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, plan.smem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(spmv_sweep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, plan.smem) !=
            cudaSuccess) {
      (void)cudaGetLastError();
      return 0;
    }
    set_bytes[d] = plan.smem;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmv_sweep_kernel<true>, 32 * SW_W, plan.smem) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
  return (int64_t)occ * sms >= (int64_t)plan.G * B;  // every range co-resident (carry handshake)
}

void launch_spmv_sweep(cudaStream_t s, const SweepPlan& plan, int n_own, const int32_t* sdesc, const int64_t* uptr,
                       const int32_t* xrun, const double* vals,
                       const double* x, double* y, double* partial, CgState* st, double* carry, unsigned* flags,
                       const BatchStrides& bs, int red_add) {
  const dim3 grid(plan.G, bs.B), block(32 * SW_W);
  static const int dbg = getenv("SSO_SWEEP_DBG") ? atoi(getenv("SSO_SWEEP_DBG")) : 0;  // timing experiments
  cudaError_t e;
  if (st)
    e = launch_cooperative_smem(spmv_sweep_kernel<true>, grid, block, (size_t)plan.smem, s, n_own, plan.L, plan.bw,
                                plan.R, sdesc, uptr, reinterpret_cast<const int2*>(xrun), vals, x, y, partial, st, carry, flags,
                                red_add, bs, dbg);
  else
    e = launch_cooperative_smem(spmv_sweep_kernel<false>, grid, block, (size_t)plan.smem, s, n_own, plan.L, plan.bw,
                                plan.R, sdesc, uptr, reinterpret_cast<const int2*>(xrun), vals, x, y, (double*)nullptr,
                                (CgState*)nullptr, carry, flags,
                                red_add, bs, dbg);
  SSO_POST_LAUNCH_RC(st ? "spmv_sweep_dot_kernel" : "spmv_sweep_kernel", e);
}

}  // namespace sso
