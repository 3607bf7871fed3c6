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
//   * consumer lane (block k, column pair B) loads the three 2x2 sub-blocks (A, B), A = 0..2,
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

#include <cfloat>
#include <cstdio>

#include "cg_common.cuh"
#include "sso_internal.h"
#include "tma.cuh"

namespace sso {

namespace {

constexpr int SW_C = 8;   // nodes per chunk
constexpr int SW_W = 6;   // consumer warps = chunk buffers
constexpr int SW_MAXU = 5, SW_MAXL = 4;

struct SweepSmem {
  static constexpr int BUF = SW_C * SW_MAXU * PULL_BLOCK;  // doubles per chunk buffer
  static constexpr int DESC = SW_C * SWEEP_DESC;           // ints per chunk descriptor copy
  static constexpr int STAGE = 2 * 6 * 16;                 // doubles per warp: 2 nodes x 6 rows x 15 lanes
  static constexpr int OWN = SW_C * 6;                     // doubles per warp: own row sums of a chunk
  static size_t bytes(int R) {
    return (size_t)SW_W * (BUF + STAGE + OWN) * 8 + (size_t)SW_W * DESC * 4 + (size_t)R * 24 * 8;
  }
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
__global__ void __launch_bounds__(32 * (SW_W + 1), 1) spmv_sweep_kernel(
    int n_own, int L, int bw, int R, const int32_t* __restrict__ sdesc, const double* __restrict__ vals,
    const double* __restrict__ p, double* __restrict__ q, double* __restrict__ partial, CgState* st,
    double* __restrict__ carry, unsigned* __restrict__ flags, int red_add, BatchStrides bs) {
  using S = SweepSmem;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[SW_W];
  __shared__ __align__(8) uint64_t desc_bar[SW_W];
  __shared__ __align__(8) uint64_t empty_bar[SW_W];
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
  carry += (int64_t)bd * G * bw * 24;
  flags += bd * G;
  const int a = r * L, b = min(n_own, a + L);
  const int nchunk = (b - a + SW_C - 1) / SW_C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* buf0 = reinterpret_cast<double*>(smem_raw);
  double* stage0 = buf0 + (size_t)SW_W * S::BUF;
  double* own0 = stage0 + (size_t)SW_W * S::STAGE;
  double* ring = own0 + (size_t)SW_W * S::OWN;  // [R][4 slots][6]
  int32_t* desc0 = reinterpret_cast<int32_t*>(ring + (size_t)R * 24);
  if (tid == 0) {
    for (int w = 0; w < SW_W; ++w) {
      mbar_init(&full_bar[w], 1);
      mbar_init(&desc_bar[w], 1);
      mbar_init(&empty_bar[w], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    done_upto = 0;
    s_epoch = *reinterpret_cast<volatile unsigned*>(flags + r);
  }
  __syncthreads();
  double pq = 0.0;
  if (warp == SW_W) {
    // ---------------- producer: descriptors + one bulk copy of the chunk's upper runs -------
    const uint64_t pol = evict_first_policy();
    for (int k = 0; k < nchunk; ++k) {
      const int w = k % SW_W;
      if (k >= SW_W) mbar_wait(&empty_bar[w], (unsigned)(((k / SW_W) - 1) & 1));
      const int first = a + k * SW_C, nc = min(SW_C, b - first);
      int32_t* D = desc0 + (size_t)w * S::DESC;
      int4 d0 = make_int4(0, 0, 0, 0);
      if (lane < nc) {
        const int4* src = reinterpret_cast<const int4*>(sdesc + SWEEP_DESC * ((int64_t)first + lane));
        int4* dst = reinterpret_cast<int4*>(D + SWEEP_DESC * lane);
        d0 = __ldg(src);
        dst[0] = d0;
        dst[1] = __ldg(src + 1);
        dst[2] = __ldg(src + 2);
        dst[3] = __ldg(src + 3);
      }
      const int b_first = __shfl_sync(FULL, d0.x, 0);
      const int b_end = __shfl_sync(FULL, d0.x + (d0.y & 255), nc - 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&desc_bar[w]);
        const unsigned bytes = (unsigned)(8 * PULL_BLOCK * (b_end - b_first));
        mbar_arrive_expect_tx(&full_bar[w], bytes);
        bulk_g2s(buf0 + (size_t)w * S::BUF, vals + PULL_BLOCK * (int64_t)b_first, bytes, &full_bar[w], pol);
      }
      __syncwarp();
    }
  } else {
    // ---------------- consumers: warp `warp` takes chunks warp, warp + W, ... ---------------
    const int w = warp;
    const double* buf = buf0 + (size_t)w * S::BUF;
    double* stage = stage0 + (size_t)w * S::STAGE;
    double* own = own0 + (size_t)w * S::OWN;
    const int32_t* D = desc0 + (size_t)w * S::DESC;
    // lane -> (node of the pass, block k, column pair B); lanes 30, 31 idle in the products
    const int ns = lane / 15, u = lane - 15 * (lane / 15), kb = u / 3, Bc = u - 3 * (u / 3);
    int offs[3];
#pragma unroll
    for (int A = 0; A < 3; ++A) offs[A] = pull_sub_off(3 * Bc + A);
    for (int k = w, it = 0; k < nchunk; k += SW_W, ++it) {
      const int first = a + k * SW_C, nc = min(SW_C, b - first);
      const unsigned ph = (unsigned)(it & 1);
      mbar_wait(&desc_bar[w], ph);
      const int b_first = D[0];
      bool waited = false;
#pragma unroll 1
      for (int pass = 0; pass < SW_C / 2; ++pass) {
        const int i = 2 * pass + ns;
        const int* Di = D + SWEEP_DESC * (i < nc ? i : 0);
        const int udeg = Di[1] & 255;
        const bool act = lane < 30 && i < nc && kb < udeg;
        double2 xm = make_double2(0.0, 0.0), xn[3];
        xn[0] = xn[1] = xn[2] = make_double2(0.0, 0.0);
        int m = 0;
        if (act) {
          m = Di[2 + kb];
          const int n = first + i;
          xm = *reinterpret_cast<const double2*>(p + 6 * (int64_t)m + 2 * Bc);
          const double2* xp = reinterpret_cast<const double2*>(p + 6 * (int64_t)n);
          xn[0] = xp[0];
          xn[1] = xp[1];
          xn[2] = xp[2];
        }
        if (!waited) {
          mbar_wait(&full_bar[w], ph);
          waited = true;
        }
        double o[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        double t0 = 0.0, t1 = 0.0;
        if (act) {
          const double* rec = buf + PULL_BLOCK * (Di[0] - b_first + kb);
#pragma unroll
          for (int A = 0; A < 3; ++A) {
            // sub-block (A, B): K[2A][2B], K[2A+1][2B], K[2A][2B+1], K[2A+1][2B+1]
            const double2 c0 = *reinterpret_cast<const double2*>(rec + offs[A]);
            const double2 c1 = *reinterpret_cast<const double2*>(rec + offs[A] + 2);
            o[2 * A] = fma(c0.x, xm.x, c1.x * xm.y);
            o[2 * A + 1] = fma(c0.y, xm.x, c1.y * xm.y);
            const double xa0 = A == 0 ? xn[0].x : (A == 1 ? xn[1].x : xn[2].x);
            const double xa1 = A == 0 ? xn[0].y : (A == 1 ? xn[1].y : xn[2].y);
            t0 = fma(c0.x, xa0, fma(c0.y, xa1, t0));
            t1 = fma(c1.x, xa0, fma(c1.y, xa1, t1));
          }
          if (kb >= 1) {
            const int slot = Di[6 + kb];
            if (slot >= 0) {
              const int rs = (m - a) % R;
              *reinterpret_cast<double2*>(ring + (size_t)rs * 24 + 6 * slot + 2 * Bc) = make_double2(t0, t1);
            }
          }
        }
        if (lane < 30) {
          double* sg = stage + ns * 96 + u;
#pragma unroll
          for (int rr = 0; rr < 6; ++rr) sg[16 * rr] = o[rr];
        }
        __syncwarp();
        if (lane < 12) {  // own row sums of the pass's two nodes: 15 partials in a fixed tree
          const int n2 = lane / 6, row = lane - 6 * (lane / 6);
          const double* sg = stage + n2 * 96 + 16 * row;
          double v[15];
#pragma unroll
          for (int j = 0; j < 15; ++j) v[j] = sg[j];
          const double s = ((((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]))) +
                            (((v[8] + v[9]) + (v[10] + v[11])) + ((v[12] + v[13]) + v[14])));
          own[6 * (2 * pass + n2) + row] = s;
        }
        __syncwarp();
      }
      if (!waited) mbar_wait(&full_bar[w], ph);
      // publish this chunk's ring contributions in chunk order
      __syncwarp();
      if (lane == 0) {
        // bounded: a broken chain reports SSO_E_CUDA instead of hanging the device
        int spin = 0;
        while (ld_acquire_cta(&done_upto) != (unsigned)k && ++spin < (1 << 22)) __nanosleep(32);
        if (spin >= (1 << 22) && DOT) {
          st->status = SSO_E_CUDA;
          st->done = 1;
        }
        st_release_cta(&done_upto, (unsigned)(k + 1));
      }
      __syncwarp();
      // every earlier chunk of the range has stored its contributions: finalise the chunk's rows
      for (int idx = lane; idx < 6 * nc; idx += 32) {
        const int i = idx / 6, row = idx - 6 * (idx / 6);
        const int* Di = D + SWEEP_DESC * i;
        const int n = first + i;
        const int ldeg = (Di[1] >> 8) & 255;
        double y = own[6 * i + row];
        const double* rg = ring + (size_t)((n - a) % R) * 24 + row;
        for (int s = 0; s < ldeg; ++s)
          if (Di[11 + s] >= a) y += rg[6 * s];
        q[6 * (int64_t)n + row] = y;
        if (DOT) pq = fma(p[6 * (int64_t)n + row], y, pq);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[w]);
    }
  }
  __syncthreads();
  // hand the contributions to the next range's first bw nodes over; take ours from the previous
  const unsigned epoch = s_epoch;
  if (r + 1 < G) {
    const int m_end = min(n_own, b + bw);
    for (int idx = tid; idx < 24 * (m_end - b); idx += blockDim.x) {
      const int mm = idx / 24, rest = idx - 24 * mm;
      carry[(int64_t)(r + 1) * bw * 24 + idx] = ring[(size_t)((b + mm - a) % R) * 24 + rest];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release_gpu(flags + r, epoch + 1);
  } else if (tid == 0) {
    st_release_gpu(flags + r, epoch + 1);
  }
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
      const double* cin = carry + (int64_t)r * bw * 24;
      for (int idx = tid; idx < 6 * (m_end - a); idx += blockDim.x) {
        const int mm = idx / 6, row = idx - 6 * mm;
        const int n = a + mm;
        const int* Dn = sdesc + SWEEP_DESC * (int64_t)n;
        const int ldeg = (Dn[1] >> 8) & 255;
        double d = 0.0;
        for (int s = 0; s < ldeg; ++s)
          if (Dn[11 + s] < a) d += cin[mm * 24 + 6 * s + row];
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
  plan.bw = bw;
  plan.R = bw + (2 * SW_W + 1) * SW_C;
  plan.smem = (int)SweepSmem::bytes(plan.R);
  if (plan.smem > 227 * 1024) return false;
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
  static uint64_t attr_mask = 0;
  int d = 0;
  cudaGetDevice(&d);
  if (!(attr_mask & (1ull << d))) {
    cudaFuncSetAttribute(spmv_sweep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(spmv_sweep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_mask |= 1ull << d;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmv_sweep_kernel<true>, 32 * (SW_W + 1), plan.smem) !=
      cudaSuccess)
    return 0;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
  return (int64_t)occ * sms >= (int64_t)plan.G * B;  // every range co-resident (carry handshake)
}

void launch_spmv_sweep(cudaStream_t s, const SweepPlan& plan, int n_own, const int32_t* sdesc, const double* vals,
                       const double* x, double* y, double* partial, CgState* st, double* carry, unsigned* flags,
                       const BatchStrides& bs, int red_add) {
  const dim3 grid(plan.G, bs.B), block(32 * (SW_W + 1));
  cudaError_t e;
  if (st)
    e = launch_cooperative_smem(spmv_sweep_kernel<true>, grid, block, (size_t)plan.smem, s, n_own, plan.L, plan.bw,
                                plan.R, sdesc, vals, x, y, partial, st, carry, flags, red_add, bs);
  else
    e = launch_cooperative_smem(spmv_sweep_kernel<false>, grid, block, (size_t)plan.smem, s, n_own, plan.L, plan.bw,
                                plan.R, sdesc, vals, x, y, (double*)nullptr, (CgState*)nullptr, carry, flags, red_add,
                                bs);
  SSO_POST_LAUNCH_RC(st ? "spmv_sweep_dot_kernel" : "spmv_sweep_kernel", e);
}

}  // namespace sso
