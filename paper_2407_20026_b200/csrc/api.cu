// C-ABI entry points (include/sso.h).  Host orchestration only: validation,
// pattern / partition build (pattern.cpp), device buffers, launch sequencing,
// the PCG chunk graphs, halo exchange + allreduce transports and the exports.
// Every step of the hot path runs in the kernels of elements.cu, assemble.cu,
// pcg.cu and grad.cu.
//
// A handle holds one or more PARTS: contiguous node strips
// with one element layer of redundant work at each strip edge, a halo of
// neighbour nodes, and per-part CG state.
//   * 1 part, 1 rank   : single-GPU path; CG chunks captured in CUDA graphs.
//   * P parts, 1 rank  : in-process partitions on one GPU (local transport:
//                        D2D halo copies, fixed-order device allreduce).  The
//                        user sees global buffers.
//   * 1 part, N ranks  : one strip per process/GPU (NCCL transport: ncclSend /
//                        ncclRecv halos, ncclAllReduce of the CG scalars).  The
//                        user passes the rank's owned slices.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "nccl.h"
#include "sso_internal.h"

using namespace sso;

namespace {

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (no link-time dependency; shares the process's
// libnccl.so.2 with torch when it is already loaded).
// ---------------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  std::string err;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) {
    api.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
    return api;
  }
#define SYM(f)                                             \
  api.f = (decltype(api.f))dlsym(lib, "nccl" #f);          \
  if (!api.f) {                                            \
    api.err = "missing nccl" #f;                           \
    return api;                                            \
  }
  SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(Send) SYM(Recv) SYM(AllReduce)
  SYM(GroupStart) SYM(GroupEnd) SYM(GetErrorString)
#undef SYM
  api.ok = true;
  return api;
}

std::string g_create_err;

}  // namespace

// ---------------------------------------------------------------------------
// One partition's device state.
// ---------------------------------------------------------------------------
struct Part {
  LocalMesh lm;
  int B = 1;            // designs in a batch (single-strip handles only)
  BatchStrides bs;
  int32_t n_nodes = 0, n_own = 0, n_beams = 0, n_quads = 0, n_own_quads = 0;
  int64_t ndof = 0, ndof_own = 0, nnz = 0, n_blocks = 0, n_staged = 0, n_slots = 0;
  HostPattern pat;
  // inputs
  double *x = nullptr, *y = nullptr, *z = nullptr;
  int32_t *beam_conn = nullptr, *quad_conn = nullptr;
  double *A = nullptr, *Iy = nullptr, *Iz = nullptr, *J = nullptr, *t = nullptr;
  double *E = nullptr, *nu = nullptr, *G = nullptr;
  uint8_t* fixed_mask = nullptr;
  // pattern
  int64_t* node_ptr = nullptr;
  int32_t* node_col = nullptr;
  int64_t* contrib_ptr = nullptr;
  int32_t* contrib = nullptr;
  int64_t* inc_ptr = nullptr;
  int32_t* inc_slot = nullptr;
  // matrix
  double *stage = nullptr, *vals = nullptr, *dinv = nullptr;
  // solver
  double *f = nullptr, *fbc = nullptr, *xs = nullptr, *r = nullptr, *p = nullptr, *q = nullptr,
         *tmp = nullptr, *gu = nullptr, *gf = nullptr;
  double* partial = nullptr;
  CgState* st = nullptr;
  DevFlags* flags = nullptr;
  unsigned int* tickets = nullptr;
  double* scal = nullptr;
  double *slot_partial = nullptr, *dxyz = nullptr, *dt = nullptr, *dt_own = nullptr, *dE = nullptr;
  // general-objective adjoint (sso_adjoint_solve / sso_grad_adjoint): primal backups,
  // and lambda (allocated on first use)
  double *ub = nullptr, *fb = nullptr, *lam = nullptr;
  // SIMP density (sso_set_density): rho, reference moduli E0 and (optional) G0 per element
  double *rho = nullptr, *E0 = nullptr, *G0 = nullptr;
  // design-dependent area loads (sso_set_area_load): local per-quad q, w and the
  // per-quad lumped value a = (q + w t) A / 4 [B][n_quads]
  double *ld_q = nullptr, *ld_w = nullptr, *ld_a = nullptr;
  // prescribed support displacements (sso_set_prescribed): b on the constrained DOFs
  // (0 elsewhere), K_full b, the CG right-hand side f - K_full b, an all-free mask
  double *pb = nullptr, *kb = nullptr, *feff = nullptr;
  uint8_t* free_mask = nullptr;
  std::vector<double> h_nu;             // host copies for sso_set_material
  std::vector<char> g_derived;          // G = E / (2 (1 + nu)) when G was not given
  // partition maps
  int32_t* block_rank = nullptr;      // quads [n_quads][16] (fused assembly; upper ranks when sym)
  int32_t* inc_rec = nullptr;         // fused assembly: [n_own][inc_pad][8] incidence records
  int inc_pad = 0;                    // max incident quads per node, rounded up to 4
  bool sym = false;                   // upper-block (symmetric) storage = pull (kept as one name)
  bool pull = false;                  // upper blocks with the one-pass pull SpMV (storage 3, 2x2 sub-block records)
  int32_t* lpull = nullptr;           // pull: (source node, upper block) per incoming block
  int32_t* pdesc = nullptr;           // pull: 16-int per-node descriptors (build_pull_desc)
  double* binv = nullptr;             // precond 1: [B][21][n_own] packed (K_nn)^-1
  double* zb = nullptr;               // precond 1: z = M^-1 r [B][ndof]
  bool cgf = false;                   // fused x / r / p update (cg_update_fused / _block_fused): one
                                      // part, full or pull storage, B <= the co-resident grid
  double* p2 = nullptr;               // cgf: the second p buffer (ping-pong)
  bool small = false;                 // cgf + small model: chunks of iterations in one persistent
                                      // kernel (cg_small.cu)
  // partitioned handles: single-reduction CG (cg_sr.cu) vectors u = M^-1 r and s = K p
  double *u_sr = nullptr, *s_sr = nullptr;
  // interior / boundary split of the owned rows: rows [bnd_lo, bnd_hi) need no halo value
  int32_t bnd_lo = 0, bnd_hi = 0;
  // Lanczos certification (lanczos.cu): CG coefficient history [B][lz_cap][2], the
  // tridiagonal scratch of the same size, the M scale per design (device bits, host value)
  double *lz_hist = nullptr, *lz_T = nullptr;
  int lz_cap = 0;
  unsigned long long* mscale_d = nullptr;
  std::vector<double> mscale_h;
  CUtensorMap pull_tmap;              // pull: [B n_ublocks][36] view of vals for the gather4 TMA
  UpperPattern up;
  int64_t* lptr = nullptr;            // pull: incoming blocks per node
  int64_t stored_blocks = 0;          // node blocks kept on the device for the owned rows
  int max_inc = 0, max_deg = 0;       // over owned nodes
  bool fused = false;                 // element + assembly in one pass (quad-only meshes)
  int32_t* own_quad_local = nullptr;  // [n_own_quads]
  int32_t* own_quad_gid = nullptr;    // [n_own_quads] global quad ids (virtual parts)
  int32_t* send_idx = nullptr;        // concatenated send lists (local owned node ids)
  double* sendbuf = nullptr;
  std::vector<int64_t> send_off;      // per neighbour, in nodes
  int64_t n_send = 0;
};

struct sso_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t cap_stream = nullptr;
  // the caller works on the legacy default stream (sso_set_stream(h, NULL, SSO_MEM_DEVICE)):
  // every entry point orders the handle's stream after it and it after the handle's work
  bool order_legacy = false;
  cudaEvent_t ev_order[2] = {nullptr, nullptr};
  sso_mem mem = SSO_MEM_HOST;
  double rtol = 1e-10;
  int64_t max_iter = 200000;
  double drill_alpha = 1e-3;
  int warm_start = 0;
  int check_every = 64;
  bool simp = false;        // sso_set_density active (E = rho^P E0)
  bool simp_chain = false;  // sso_grad_density in progress: dC/dE -> dC/drho before the copy-out
  double penal = 1.0;
  int batch = 1;  // designs per handle
  int reliable = 1;  // 0 plain CG, 1 final true-residual restart, 2 + periodic replacement
  int assembly = 0;  // 0 auto (fused when the mesh allows), 1 staged
  int storage = 0;   // 1 full CSR storage, 3 upper blocks + pull SpMV (0 = 3)
  int precond = 0;   // 0 point Jacobi, 1 node-block Jacobi (block_jacobi.cu)
  bool area_load = false;  // design-dependent area loads active (sso_set_area_load)
  bool skip_load = false;  // adjoint solves: the right-hand side is dg/du only, b = 0
  bool prescribed = false; // non-zero support displacements active (sso_set_prescribed)
  double ld_dir[3] = {0.0, 0.0, 0.0};

  // global problem sizes and what this handle's user buffers cover
  int32_t g_nodes = 0, g_beams = 0, g_quads = 0;
  int32_t user_node_begin = 0, user_nodes = 0, user_quads = 0;
  int nranks = 1, rank = 0;
  ncclComm_t comm = nullptr;
  std::vector<std::unique_ptr<Part>> parts;
  CgState** d_sts = nullptr;   // device array of the parts' CgState pointers
  // in-process halo fill (one launch for all parts): entries (dst part, dst node, src part,
  // src node) and, per vector kind, the device array of the parts' base pointers
  int4* d_halo_ent = nullptr;
  int n_halo_ent = 0;
  double** d_vbase[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  bool split = false;          // overlap the halo exchange with the interior rows' SpMV
  cudaStream_t side_stream = nullptr;  // halo exchange stream during capture (split)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // in-process parts: one stream per part inside the captured iterations, so the parts'
  // SpMVs and updates overlap (one part's tail with the next part's start)
  std::vector<cudaStream_t> part_streams;
  std::vector<cudaEvent_t> part_ev;
  // in-process parts in ONE launch per step (grid.y = part): device arrays of per-part
  // operands for the pull SpMV (u -> q) and the single-reduction update
  PullPart* d_pull_parts = nullptr;
  SrPart* d_sr_parts = nullptr;
  int max_own = 0;
  double* d_dt_all = nullptr;  // virtual parts: global dC/dt assembly buffer
  double* h_C = nullptr;       // pinned scalar

  CgState* h_st = nullptr;
  CgState* h_chunk = nullptr;  // [2]
  DevFlags* h_flags = nullptr;
  double* h_scal = nullptr;
  unsigned long long* h_mscale = nullptr;  // [parts][batch] pinned: the assembly's m_min bits
  bool mscale_pending = false;             // h_mscale written by the stream, not yet read

  bool assembled = false, solved = false;
  cudaGraphExec_t chunk_exec = nullptr;
  cudaGraphExec_t prof_exec[2] = {nullptr, nullptr};
  long long kernels_per_chunk = 0;
  std::vector<cudaEvent_t> chunk_ev[2];
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_done[2] = {nullptr, nullptr};

  // hat filter neighbour grids (sso_hat_filter), one per point kind, rebuilt when the
  // radius or the geometry changes
  struct FilterGrid {
    bool valid = false;
    double radius = 0.0;
    int32_t n = 0;
    int gx = 1, gy = 1, gz = 1;
    double *px = nullptr, *py = nullptr, *pz = nullptr, *io = nullptr;  // io: [2][3][n] host-mem staging
    int32_t *cell_of = nullptr, *perm = nullptr;
    int64_t* cell_start = nullptr;
  } fgrid[2];

  Timers tm;
  long long launches = 0;
  std::string err;

  // NCCL transport: every multi-rank handle; a 1-rank handle with a unique id when
  // SSO_NCCL_SELF=1 (tests: the whole NCCL path -- comm, captured allreduces, the split --
  // on one GPU with no peer to wait for)
  bool use_nccl = false;
  bool distributed() const { return parts.size() > 1 || use_nccl; }
  Part& P0() { return *parts[0]; }
};

#define FAIL(h, code, msg) \
  do {                     \
    (h)->err = (msg);      \
    return (code);         \
  } while (0)

#define CK(h, call)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      (h)->err = std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call; \
      return e_ == cudaErrorMemoryAllocation ? SSO_E_OOM : SSO_E_CUDA;                \
    }                                                                                 \
  } while (0)

#define CKL(h)                                                                       \
  do {                                                                               \
    cudaError_t e_ = cudaGetLastError();                                             \
    if (e_ != cudaSuccess) {                                                         \
      (h)->err = std::string("CUDA launch error: ") + cudaGetErrorString(e_) + " (" + \
                 last_launch_error() + ")";                                          \
      return SSO_E_CUDA;                                                             \
    }                                                                                \
  } while (0)

#define CKN(h, call)                                                                     \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) {                                                             \
      (h)->err = std::string("NCCL error: ") + nccl().GetErrorString(r_) + " at " #call; \
      return SSO_E_NCCL;                                                                 \
    }                                                                                    \
  } while (0)

namespace {

template <class T>
int dalloc(sso_ctx* h, T** p, int64_t n) {
  if (n <= 0) n = 1;
  cudaError_t e = cudaMalloc((void**)p, (size_t)n * sizeof(T));
  if (e != cudaSuccess) {
    h->err = std::string("cudaMalloc failed (") + std::to_string((size_t)n * sizeof(T)) +
             " bytes): " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? SSO_E_OOM : SSO_E_CUDA;
  }
  return SSO_OK;
}

template <class T>
int upload(sso_ctx* h, T** p, const T* src, int64_t n) {
  int rc = dalloc(h, p, n);
  if (rc) return rc;
  if (n > 0 && src) CK(h, cudaMemcpy(*p, src, (size_t)n * sizeof(T), cudaMemcpyHostToDevice));
  return SSO_OK;
}

cudaMemcpyKind kind_in(const sso_ctx* h) {
  return h->mem == SSO_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
}
cudaMemcpyKind kind_out(const sso_ctx* h) {
  return h->mem == SSO_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
}

bool finite_all(const double* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

// --- timers ---------------------------------------------------------------
cudaEvent_t pool_event(sso_ctx* h) {
  Timers& T = h->tm;
  if (T.pool_used == T.pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    T.pool.push_back(e);
  }
  return T.pool[T.pool_used++];
}

struct Scope {
  sso_ctx* h;
  int fam;
  cudaEvent_t a = nullptr, b = nullptr;
  long long g0;
  Scope(sso_ctx* h_, int fam_) : h(h_), fam(fam_), g0(g_launches) {
    if (h->tm.on) {
      a = pool_event(h);
      b = pool_event(h);
      cudaEventRecord(a, h->stream);
    }
  }
  ~Scope() {
    h->launches += g_launches - g0;
    if (h->tm.on) {
      cudaEventRecord(b, h->stream);
      h->tm.pending.push_back({fam, {a, b}});
    }
  }
};

void flush_timers(sso_ctx* h) {
  Timers& T = h->tm;
  for (auto& pe : T.pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, pe.second.first, pe.second.second) == cudaSuccess) {
      T.total_ms[pe.first] += ms;
      T.launches[pe.first] += 1;
    } else {
      (void)cudaGetLastError();  // never leave a timing failure pending for a later check
    }
  }
  T.pending.clear();
  T.pool_used = 0;
}

int sync(sso_ctx* h) {
  CK(h, cudaStreamSynchronize(h->stream));
  flush_timers(h);
  return SSO_OK;
}

// Every ABI entry point taking a handle: make the handle's device current (restored on
// return) and, when the caller's device buffers are ordered by the legacy default stream,
// order the handle's stream after the work already queued there and that stream after
// the handle's work.
struct Entry {
  sso_ctx* h;
  int prev = -1;
  explicit Entry(sso_ctx* h_) : h(h_) {
    if (!h) return;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != h->device && cudaSetDevice(h->device) == cudaSuccess) prev = cur;
    if (h->order_legacy && h->mem == SSO_MEM_DEVICE && h->ev_order[0]) {
      cudaEventRecord(h->ev_order[0], cudaStreamLegacy);
      cudaStreamWaitEvent(h->stream, h->ev_order[0], 0);
    }
  }
  ~Entry() {
    if (!h) return;
    if (h->order_legacy && h->mem == SSO_MEM_DEVICE && h->ev_order[1]) {
      cudaEventRecord(h->ev_order[1], h->stream);
      cudaStreamWaitEvent(cudaStreamLegacy, h->ev_order[1], 0);
    }
    if (prev >= 0) cudaSetDevice(prev);
  }
};
#define ENTER(h) Entry entry_guard_(h)

// NVTX range per ABI call and per solve phase (SURVEY.md §5 "Tracing"): free without a tool
// attached (NVTX v3 is header-only; the ranges show in nsys / ncu timelines).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define TRACE(name) NvtxRange nvtx_range_(name)

// ---------------------------------------------------------------------------
// Transports: halo exchange of a per-part vector and allreduce of CgState::red.
// ---------------------------------------------------------------------------
enum VecId { V_P = 0, V_X = 1, V_GU = 2, V_TMP = 3, V_U = 4 };

double* vec_of(Part& P, int v) {
  switch (v) {
    case V_P: return P.p;
    case V_X: return P.xs;
    case V_GU: return P.gu;
    case V_U: return P.u_sr;
    default: return P.tmp;
  }
}

// y = K x for the part's owned rows (full or upper-block storage); with st also
// p^T q (and alpha, unless the fused update forms it).  x must have its halo filled
// (partitioned handles).
void spmv_apply(cudaStream_t s, Part& P, const double* x, double* y, CgState* st) {
  if (P.pull)
    launch_spmv_pull(s, &P.pull_tmap, P.n_own, (int)(P.bs.nnz / PULL_BLOCK), P.pdesc, P.node_col, P.lpull, P.vals, x, y,
                     st ? P.partial : nullptr, st, P.bs);
  else if (st)
    launch_spmv_dot(s, P.n_own, P.node_ptr, P.node_col, P.vals, x, y, P.partial, st, P.bs);
  else
    launch_spmv(s, P.n_own, P.node_ptr, P.node_col, P.vals, x, y, P.bs);
}

int exchange(sso_ctx* h, int v, cudaStream_t s = nullptr) {
  if (!h->distributed()) return SSO_OK;
  if (!s) s = h->stream;
  long long g0 = g_launches;
  if (h->use_nccl) {
    Part& P = h->P0();
    launch_pack(s, (int)P.n_send, P.send_idx, vec_of(P, v), P.sendbuf);
  }
  if (!h->use_nccl) {
    // local transport: one gather kernel fills every part's halo from its neighbours' owned rows
    launch_halo_gather(s, h->n_halo_ent, h->d_halo_ent, h->d_vbase[v]);
  } else {
    Part& P = h->P0();
    double* dst = vec_of(P, v);
    CKN(h, nccl().GroupStart());
    for (size_t k = 0; k < P.lm.nbrs.size(); ++k) {
      const NeighborPlan& nb = P.lm.nbrs[k];
      if (!nb.send_local.empty())
        CKN(h, nccl().Send(P.sendbuf + 6 * P.send_off[k], 6 * nb.send_local.size(), ncclDouble, nb.part,
                           h->comm, s));
      if (nb.recv_count)
        CKN(h, nccl().Recv(dst + 6 * ((int64_t)P.n_own + nb.recv_offset), (size_t)6 * nb.recv_count,
                           ncclDouble, nb.part, h->comm, s));
    }
    CKN(h, nccl().GroupEnd());
  }
  h->launches += g_launches - g0;
  return SSO_OK;
}

int allreduce(sso_ctx* h, int nvals, cudaStream_t s = nullptr) {
  if (!h->distributed()) return SSO_OK;
  if (!s) s = h->stream;
  long long g0 = g_launches;
  if (!h->use_nccl) {
    launch_allreduce_parts(s, h->d_sts, (int)h->parts.size(), nvals);
  } else {
    double* red = h->P0().st->red;
    CKN(h, nccl().AllReduce(red, red, nvals, ncclDouble, ncclSum, h->comm, s));
  }
  h->launches += g_launches - g0;
  return SSO_OK;
}

int check_flags(sso_ctx* h) {
  for (auto& pp : h->parts) {
    Part& P = *pp;
    // every design's flags in one copy and one synchronisation
    CK(h, cudaMemcpyAsync(h->h_flags, P.flags, P.B * sizeof(DevFlags), cudaMemcpyDeviceToHost, h->stream));
    int rc = sync(h);
    if (rc) return rc;
    for (int bd = 0; bd < P.B; ++bd) {
      const DevFlags& F = h->h_flags[bd];
      const std::string dsg = P.B > 1 ? " in design " + std::to_string(bd) : std::string();
      if (F.degenerate_elem != INT_MAX) {
        const int e = F.degenerate_elem;
        const bool beam = e < P.n_beams;
        const int g = beam ? P.lm.beam_gid[e] : P.lm.quad_gid[e - P.n_beams];
        char buf[256];
        snprintf(buf, sizeof buf, "degenerate element %d (%s %d): zero length / zero normal / det J <= 0",
                 beam ? g : h->g_beams + g, beam ? "beam" : "quad", g);
        h->err = buf + dsg;
        return SSO_E_DEGENERATE;
      }
      if (F.singular_dof != INT_MAX) {
        const int d = F.singular_dof;
        const int gnode = P.lm.node_gid[d / 6];
        char buf[256];
        snprintf(buf, sizeof buf, "singular: free DOF %d (node %d, component %d) has diagonal <= 0",
                 6 * gnode + d % 6, gnode, d % 6);
        h->err = buf + dsg;
        return SSO_E_SINGULAR;
      }
    }
  }
  return SSO_OK;
}

__global__ void reset_flags_kernel(DevFlags* flags, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[i] = DevFlags{INT_MAX, INT_MAX};
}

// the device error flags back to "none", stream-ordered (no host round trip)
int reset_flags(sso_ctx* h) {
  for (auto& pp : h->parts) {
    reset_flags_kernel<<<(pp->B + 127) / 128, 128, 0, h->stream>>>(pp->flags, pp->B);
    SSO_POST_LAUNCH("reset_flags_kernel");
  }
  return SSO_OK;
}

// Capture K = check_every CG iterations of the single-part solver into a graph.
// prof_slot >= 0 adds external event-record nodes around every PROF_EVERY-th
// SpMV (events of that slot): a live sample of the SpMV launch duration.
constexpr int PROF_EVERY = 16;

// One CG iteration on stream s (captured into the chunk graphs), ordered
// p update -> SpMV -> x / r update so that residual replacements between chunks
// land before p is formed (init sets p = z and beta = 0, so the first p update is
// a no-op).  Single part: alpha / beta are formed by the kernels' last CTAs.
// Partitioned: p update, halo of p, SpMV + local p^T q, allreduce, alpha; update +
// local r^T z / r^T r, allreduce, beta and the convergence test.  `rec` brackets part 0's SpMV with
// the event pair ev[0], ev[1].
int cg_iteration(sso_ctx* h, cudaStream_t s, const cudaEvent_t* ev, int it) {
  int rc;
  if (!h->distributed()) {
    Part& P = h->P0();
    if (P.cgf) {  // SpMV of the current p, then x / r / p_next in one kernel (ping-pong p)
      double* pc = (it & 1) ? P.p2 : P.p;
      double* pn = (it & 1) ? P.p : P.p2;
      if (ev) cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal);
      spmv_apply(s, P, pc, P.q, P.st);
      if (ev) cudaEventRecordWithFlags(ev[1], s, cudaEventRecordExternal);
      if (P.binv)
        launch_cg_update_block_fused(s, P.n_own, P.binv, P.xs, P.r, pc, P.q, pn, P.partial, P.st, P.bs);
      else
        launch_cg_update_fused(s, (int)P.ndof_own, P.dinv, P.xs, P.r, pc, P.q, pn, P.partial, P.st, P.bs);
      return SSO_OK;
    }
    if (P.binv)
      launch_cg_pupdate_z(s, (int)P.ndof_own, P.zb, P.p, P.st, P.bs);
    else
      launch_cg_pupdate(s, (int)P.ndof_own, P.dinv, P.r, P.p, P.st, P.bs);
    if (ev) cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal);
    spmv_apply(s, P, P.p, P.q, P.st);
    if (ev) cudaEventRecordWithFlags(ev[1], s, cudaEventRecordExternal);
    if (P.binv)
      launch_cg_update_block(s, P.n_own, P.binv, P.xs, P.r, P.p, P.q, P.zb, P.partial, P.st, P.bs);
    else
      launch_cg_update(s, (int)P.ndof_own, P.dinv, P.xs, P.r, P.p, P.q, P.partial, P.st, P.bs);
    return SSO_OK;
  }
  // Partitioned: single-reduction CG (cg_sr.cu).  halo of u -> w = K u (+ local delta) ->
  // one allreduce of (delta, gamma, r^T r, |f|^2) -> x / r / u / p / s update.  With the split,
  // the halo travels on the side stream while the rows that need no halo value run.
  if (h->split) {
    CK(h, cudaEventRecord(h->ev_fork, s));
    CK(h, cudaStreamWaitEvent(h->side_stream, h->ev_fork, 0));
    if ((rc = exchange(h, V_U, h->side_stream))) return rc;
    CK(h, cudaEventRecord(h->ev_join, h->side_stream));
    if (ev) cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal);
    // the u^T w pieces add up in launch order; the first piece that runs writes (empty pieces
    // launch nothing)
    for (auto& pp : h->parts) {
      Part& P = *pp;
      launch_spmv_pull(s, &P.pull_tmap, P.bnd_hi, (int)(P.bs.nnz / PULL_BLOCK), P.pdesc, P.node_col, P.lpull,
                       P.vals, P.u_sr, P.q, P.partial, P.st, P.bs, P.bnd_lo, 0);
    }
    CK(h, cudaStreamWaitEvent(s, h->ev_join, 0));
    for (auto& pp : h->parts) {
      Part& P = *pp;
      const bool mid = P.bnd_hi > P.bnd_lo, lo = P.bnd_lo > 0;
      launch_spmv_pull(s, &P.pull_tmap, P.bnd_lo, (int)(P.bs.nnz / PULL_BLOCK), P.pdesc, P.node_col, P.lpull,
                       P.vals, P.u_sr, P.q, P.partial, P.st, P.bs, 0, mid ? 1 : 0);
      launch_spmv_pull(s, &P.pull_tmap, P.n_own, (int)(P.bs.nnz / PULL_BLOCK), P.pdesc, P.node_col, P.lpull,
                       P.vals, P.u_sr, P.q, P.partial, P.st, P.bs, P.bnd_hi, (mid || lo) ? 1 : 0);
    }
    if (ev) cudaEventRecordWithFlags(ev[1], s, cudaEventRecordExternal);
  } else {
    if ((rc = exchange(h, V_U, s))) return rc;
    if (h->d_pull_parts) {  // every part's SpMV in one launch
      if (ev) cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal);
      launch_spmv_pull_multi(s, h->d_pull_parts, (int)h->parts.size(), h->max_own);
      if (ev) cudaEventRecordWithFlags(ev[1], s, cudaEventRecordExternal);
    } else if (!h->part_streams.empty() && !ev) {
      // in-process parts: the parts' SpMVs on their own streams (fork / join inside the graph)
      const size_t np = h->parts.size();
      CK(h, cudaEventRecord(h->ev_fork, s));
      for (size_t i = 0; i < np; ++i) {
        Part& P = *h->parts[i];
        CK(h, cudaStreamWaitEvent(h->part_streams[i], h->ev_fork, 0));
        if (P.pull)  // each part on 1/np of the persistent grid: the parts run side by side
          launch_spmv_pull(h->part_streams[i], &P.pull_tmap, P.n_own, (int)(P.bs.nnz / PULL_BLOCK), P.pdesc,
                           P.node_col, P.lpull, P.vals, P.u_sr, P.q, P.partial, P.st, P.bs, 0, 0, (int)np);
        else
          spmv_apply(h->part_streams[i], P, P.u_sr, P.q, P.st);
        CK(h, cudaEventRecord(h->part_ev[i], h->part_streams[i]));
      }
      for (size_t i = 0; i < np; ++i) CK(h, cudaStreamWaitEvent(s, h->part_ev[i], 0));
    } else {
      bool first = true;
      for (auto& pp : h->parts) {
        Part& P = *pp;
        if (ev && first) cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal);
        spmv_apply(s, P, P.u_sr, P.q, P.st);
        if (ev && first) cudaEventRecordWithFlags(ev[1], s, cudaEventRecordExternal);
        first = false;
      }
    }
  }
  if ((rc = allreduce(h, 4, s))) return rc;
  if (h->d_sr_parts) {
    launch_cgsr_update_multi(s, h->d_sr_parts, (int)h->parts.size(), h->max_own);
    return SSO_OK;
  }
  if (!h->part_streams.empty()) {
    const size_t np = h->parts.size();
    CK(h, cudaEventRecord(h->ev_fork, s));
    for (size_t i = 0; i < np; ++i) {
      Part& P = *h->parts[i];
      CK(h, cudaStreamWaitEvent(h->part_streams[i], h->ev_fork, 0));
      launch_cgsr_update(h->part_streams[i], P.n_own, P.dinv, P.binv, P.xs, P.r, P.u_sr, P.q, P.p, P.s_sr,
                         P.partial, P.st, (int)np);
      CK(h, cudaEventRecord(h->part_ev[i], h->part_streams[i]));
    }
    for (size_t i = 0; i < np; ++i) CK(h, cudaStreamWaitEvent(s, h->part_ev[i], 0));
    return SSO_OK;
  }
  for (auto& pp : h->parts) {
    Part& P = *pp;
    launch_cgsr_update(s, P.n_own, P.dinv, P.binv, P.xs, P.r, P.u_sr, P.q, P.p, P.s_sr, P.partial, P.st);
  }
  return SSO_OK;
}

int build_chunk_graph(sso_ctx* h, int prof_slot, cudaGraphExec_t* out) {
  if (*out) {
    cudaGraphExecDestroy(*out);
    *out = nullptr;
  }
  const int K = h->check_every;
  if (prof_slot >= 0) {
    auto& ev = h->chunk_ev[prof_slot];
    while ((int)ev.size() < 2 * K) {
      cudaEvent_t e;
      CK(h, cudaEventCreate(&e));
      ev.push_back(e);
    }
  }
  long long g0 = g_launches, l0 = h->launches;
  CK(h, cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
  int rc = SSO_OK;
  if (!h->distributed() && h->P0().small) {  // the whole chunk in one persistent kernel
    Part& P = h->P0();
    // 4 chunks' worth of iterations per launch (the kernel stops at convergence) unless periodic
    // residual replacements need the chunk boundaries: fewer launches and state polls
    const int iters = h->reliable >= 2 ? K : 4 * K;
    launch_cg_small(h->cap_stream, P.n_own, iters, P.pdesc, P.vals, P.dinv, P.xs, P.r, P.p, P.p2, P.st, P.bs);
  } else {
    for (int i = 0; i < K && rc == SSO_OK; ++i) {
      const bool rec = prof_slot >= 0 && (i % PROF_EVERY) == 0;
      rc = cg_iteration(h, h->cap_stream, rec ? &h->chunk_ev[prof_slot][2 * i] : nullptr, i);
    }
  }
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
  // every kernel bumps g_launches once (exchange / allreduce also add to h->launches):
  // undo both and count the chunk's kernels per replay instead
  h->kernels_per_chunk = g_launches - g0;
  h->launches = l0;
  g_launches = g0;
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) {
    h->err = std::string("graph capture failed: ") + cudaGetErrorString(e);
    return SSO_E_CUDA;
  }
  e = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    h->err = std::string("graph instantiate failed: ") + cudaGetErrorString(e);
    return SSO_E_CUDA;
  }
  return SSO_OK;
}

void free_part(Part& P) {
  void* ptrs[] = {P.x, P.y, P.z, P.beam_conn, P.quad_conn, P.A, P.Iy, P.Iz, P.J, P.t, P.E, P.nu, P.G,
                  P.fixed_mask, P.node_ptr, P.node_col, P.contrib_ptr, P.contrib, P.inc_ptr,
                  P.inc_slot, P.stage, P.vals, P.dinv, P.f, P.fbc, P.xs, P.r, P.p, P.q, P.tmp, P.gu,
                  P.gf, P.partial, P.st, P.flags, P.tickets, P.scal, P.slot_partial, P.dxyz, P.dt,
                  P.dt_own, P.own_quad_local, P.own_quad_gid, P.send_idx, P.sendbuf, P.block_rank,
                  P.lptr, P.lpull, P.pdesc, P.binv, P.zb, P.p2, P.dE,
                  P.ub, P.fb, P.inc_rec, P.lam, P.ld_q, P.ld_w, P.ld_a, P.pb, P.kb, P.feff, P.free_mask,
                  P.rho, P.E0, P.G0, P.lz_hist, P.lz_T, P.mscale_d, P.u_sr, P.s_sr};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}

void free_filter_grid(sso_ctx::FilterGrid& g) {
  void* ptrs[] = {g.px, g.py, g.pz, g.io, g.cell_of, g.perm, g.cell_start};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  g = sso_ctx::FilterGrid();
}

void free_all(sso_ctx* h) {
  for (auto& g : h->fgrid) free_filter_grid(g);
  for (auto& pp : h->parts) free_part(*pp);
  h->parts.clear();
  if (h->d_sts) cudaFree(h->d_sts);
  if (h->d_halo_ent) cudaFree(h->d_halo_ent);
  if (h->d_pull_parts) cudaFree(h->d_pull_parts);
  if (h->d_sr_parts) cudaFree(h->d_sr_parts);
  for (auto b : h->d_vbase)
    if (b) cudaFree(b);
  if (h->side_stream) cudaStreamDestroy(h->side_stream);
  for (auto ps : h->part_streams)
    if (ps) cudaStreamDestroy(ps);
  for (auto e : h->part_ev)
    if (e) cudaEventDestroy(e);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->d_dt_all) cudaFree(h->d_dt_all);
  if (h->h_C) cudaFreeHost(h->h_C);
  if (h->h_st) cudaFreeHost(h->h_st);
  if (h->h_chunk) cudaFreeHost(h->h_chunk);
  if (h->h_scal) cudaFreeHost(h->h_scal);
  if (h->h_flags) cudaFreeHost(h->h_flags);
  if (h->h_mscale) cudaFreeHost(h->h_mscale);
  if (h->chunk_exec) cudaGraphExecDestroy(h->chunk_exec);
  for (int k = 0; k < 2; ++k) {
    if (h->prof_exec[k]) cudaGraphExecDestroy(h->prof_exec[k]);
    for (auto e : h->chunk_ev[k]) cudaEventDestroy(e);
  }
  for (auto e : h->tm.pool) cudaEventDestroy(e);
  if (h->ev_a) cudaEventDestroy(h->ev_a);
  if (h->ev_b) cudaEventDestroy(h->ev_b);
  for (auto e : h->ev_done)
    if (e) cudaEventDestroy(e);
  for (auto e : h->ev_order)
    if (e) cudaEventDestroy(e);
  if (h->comm && nccl().ok) nccl().CommDestroy(h->comm);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
}

int validate(const sso_mesh* m, const sso_sections* s, const sso_materials* mt,
             const sso_supports* sp, std::string& err) {
  char buf[256];
  if (!m || !s || !mt || !sp) { err = "null argument"; return SSO_E_INVALID; }
  if (m->n_nodes <= 0 || !m->x || !m->y || !m->z) { err = "mesh: n_nodes <= 0 or null coordinates"; return SSO_E_INVALID; }
  if (m->n_beams < 0 || m->n_quads < 0 || m->n_beams + m->n_quads == 0) { err = "mesh: no elements"; return SSO_E_INVALID; }
  if ((int64_t)m->n_nodes * 6 > INT_MAX) { err = "mesh: too many nodes for int32 DOF indices"; return SSO_E_INVALID; }
  if (m->n_beams > 0 && (!m->beam_conn || !s->A || !s->Iy || !s->Iz || !s->J)) { err = "beams: null connectivity or section"; return SSO_E_INVALID; }
  if (m->n_quads > 0 && (!m->quad_conn || !s->t)) { err = "quads: null connectivity or thickness"; return SSO_E_INVALID; }
  if (!mt->E || !mt->nu) { err = "materials: null E or nu"; return SSO_E_INVALID; }
  const int64_t ne = (int64_t)m->n_beams + m->n_quads;
  if (!finite_all(m->x, m->n_nodes) || !finite_all(m->y, m->n_nodes) || !finite_all(m->z, m->n_nodes)) { err = "mesh: non-finite coordinate"; return SSO_E_INVALID; }
  for (int64_t e = 0; e < ne; ++e) {
    const double E = mt->E[e], nu = mt->nu[e];
    if (!(E > 0.0) || !std::isfinite(E)) { snprintf(buf, sizeof buf, "element %lld: E <= 0 or non-finite", (long long)e); err = buf; return SSO_E_INVALID; }
    if (!(nu >= 0.0 && nu < 0.5)) { snprintf(buf, sizeof buf, "element %lld: nu outside [0, 0.5)", (long long)e); err = buf; return SSO_E_INVALID; }
    if (mt->G && (!(mt->G[e] > 0.0) || !std::isfinite(mt->G[e]))) { snprintf(buf, sizeof buf, "element %lld: G <= 0", (long long)e); err = buf; return SSO_E_INVALID; }
  }
  for (int32_t e = 0; e < m->n_beams; ++e) {
    const int32_t a = m->beam_conn[2 * e], b = m->beam_conn[2 * e + 1];
    if (a < 0 || a >= m->n_nodes || b < 0 || b >= m->n_nodes) { snprintf(buf, sizeof buf, "beam %d: node index out of range", e); err = buf; return SSO_E_INVALID; }
    if (a == b) { snprintf(buf, sizeof buf, "beam %d: i_node == j_node", e); err = buf; return SSO_E_INVALID; }
    const double v[4] = {s->A[e], s->Iy[e], s->Iz[e], s->J[e]};
    for (double vv : v)
      if (!(vv > 0.0) || !std::isfinite(vv)) { snprintf(buf, sizeof buf, "beam %d: A, Iy, Iz or J <= 0", e); err = buf; return SSO_E_INVALID; }
    const double dx = m->x[b] - m->x[a], dy = m->y[b] - m->y[a], dz = m->z[b] - m->z[a];
    if (!(dx * dx + dy * dy + dz * dz > 0.0)) { snprintf(buf, sizeof buf, "degenerate element %d (beam): zero length", e); err = buf; return SSO_E_DEGENERATE; }
  }
  for (int32_t q = 0; q < m->n_quads; ++q) {
    const int32_t* c = m->quad_conn + 4 * (int64_t)q;
    for (int i = 0; i < 4; ++i) {
      if (c[i] < 0 || c[i] >= m->n_nodes) { snprintf(buf, sizeof buf, "quad %d: node index out of range", q); err = buf; return SSO_E_INVALID; }
      for (int j = 0; j < i; ++j)
        if (c[i] == c[j]) { snprintf(buf, sizeof buf, "quad %d: repeated node %d", q, c[i]); err = buf; return SSO_E_INVALID; }
    }
    if (!(s->t[q] > 0.0) || !std::isfinite(s->t[q])) { snprintf(buf, sizeof buf, "quad %d: t <= 0", q); err = buf; return SSO_E_INVALID; }
  }
  if (sp->n <= 0 || !sp->node || !sp->mask6) { err = "supports: none given (the structure would be singular)"; return SSO_E_INVALID; }
  for (int32_t k = 0; k < sp->n; ++k) {
    if (sp->node[k] < 0 || sp->node[k] >= m->n_nodes) { snprintf(buf, sizeof buf, "support %d: node out of range", k); err = buf; return SSO_E_INVALID; }
    if ((sp->mask6[k] & 63) == 0) { snprintf(buf, sizeof buf, "support %d: all-zero mask", k); err = buf; return SSO_E_INVALID; }
  }
  return SSO_OK;
}

std::vector<int32_t> make_ranges(int32_t n_nodes, int32_t n_parts, const int32_t* given) {
  std::vector<int32_t> r((size_t)n_parts + 1);
  if (given) {
    for (int32_t p = 0; p <= n_parts; ++p) r[p] = given[p];
  } else {
    for (int32_t p = 0; p <= n_parts; ++p) r[p] = (int32_t)(((int64_t)n_nodes * p) / n_parts);
  }
  return r;
}

// Build one part's device state from the (validated) global inputs.
int setup_part(sso_ctx* h, Part& P, const sso_mesh* mesh, const sso_sections* sec,
               const sso_materials* mat, const std::vector<uint8_t>& gmask,
               const std::vector<double>& gG) {
  const LocalMesh& L = P.lm;
  P.n_nodes = (int32_t)L.node_gid.size();
  P.n_own = L.n_own;
  P.n_beams = (int32_t)L.beam_gid.size();
  P.n_quads = (int32_t)L.quad_gid.size();
  P.n_own_quads = (int32_t)L.own_quad_local.size();
  P.ndof = 6 * (int64_t)P.n_nodes;
  P.ndof_own = 6 * (int64_t)P.n_own;
  std::string perr = build_pattern(P.n_nodes, P.n_beams, L.beam_conn.data(), P.n_quads,
                                   L.quad_conn.data(), P.pat);
  if (!perr.empty()) { h->err = perr; return SSO_E_INVALID; }
  P.n_blocks = P.pat.n_blocks();
  P.n_staged = P.pat.n_staged_blocks();
  P.n_slots = 2 * (int64_t)P.n_beams + 4 * (int64_t)P.n_quads;
  P.nnz = 36 * (P.pat.node_ptr[P.n_own]);  // owned rows only
  for (int32_t n = 0; n < P.n_own; ++n) {
    P.max_inc = std::max<int>(P.max_inc, (int)(P.pat.inc_ptr[n + 1] - P.pat.inc_ptr[n]));
    P.max_deg = std::max<int>(P.max_deg, (int)(P.pat.node_ptr[n + 1] - P.pat.node_ptr[n]));
  }
  P.fused = h->assembly == 0 && P.n_beams == 0 && P.n_quads > 0 && P.max_deg <= fused_max_degree();
  // Storage 3 works on strips too: owned nodes come first in the local numbering, so every
  // lower neighbour (n < m) of an owned row m is owned and stores the block (n, m) itself, and
  // halo neighbours are always upper.
  P.sym = P.pull = (h->storage == 3);
  if (P.pull && P.pat.node_ptr[P.n_nodes] >= INT32_MAX / PULL_BLOCK) {  // 32-bit offsets in the pull kernel
    h->err = "storage 3: too many node blocks for 32-bit offsets";
    return SSO_E_INVALID;
  }
  // the pull descriptor packs a node's degree in 8 bits: a node with more than 255
  // neighbours (a large beam fan) keeps the whole strip on full storage
  for (int32_t n = 0; P.pull && n < P.n_nodes; ++n)
    if (P.pat.node_ptr[n + 1] - P.pat.node_ptr[n] > 255) P.sym = P.pull = false;
  if (P.sym) build_upper(P.pat, L.beam_conn.data(), L.quad_conn.data(), P.up);
  P.stored_blocks = P.sym ? P.up.uptr[P.n_own] : P.pat.node_ptr[P.n_own];
  const int64_t ne = (int64_t)P.n_beams + P.n_quads;
  const int B = P.B = h->batch;
  P.bs.B = B;
  P.bs.node = P.n_nodes;
  P.bs.quad = P.n_quads;
  P.bs.stage = 36 * P.n_staged;
  P.bs.nnz = P.pull ? PULL_BLOCK * P.up.n_ublocks() : 36 * (P.sym ? P.up.n_ublocks() : P.n_blocks);
  P.bs.dof = P.ndof;
  P.bs.partial = 16 * (int64_t)cg_grid();
  P.bs.slot = 3 * std::max<int64_t>(P.n_slots, 1);
  // per-design arrays start as B copies of the given design (sso_set_design replaces them)
  std::vector<double> x((size_t)B * P.n_nodes), y((size_t)B * P.n_nodes), z((size_t)B * P.n_nodes);
  std::vector<uint8_t> mask(P.n_nodes);
  for (int32_t i = 0; i < P.n_nodes; ++i) {
    const int32_t g = L.node_gid[i];
    for (int b = 0; b < B; ++b) {
      x[(size_t)b * P.n_nodes + i] = mesh->x[g];
      y[(size_t)b * P.n_nodes + i] = mesh->y[g];
      z[(size_t)b * P.n_nodes + i] = mesh->z[g];
    }
    mask[i] = gmask[g];
  }
  std::vector<double> A(P.n_beams), Iy(P.n_beams), Iz(P.n_beams), Jt(P.n_beams), t((size_t)B * P.n_quads);
  std::vector<double> E(ne), nu(ne), G(ne);
  for (int32_t k = 0; k < P.n_beams; ++k) {
    const int32_t g = L.beam_gid[k];
    A[k] = sec->A[g];
    Iy[k] = sec->Iy[g];
    Iz[k] = sec->Iz[g];
    Jt[k] = sec->J[g];
    E[k] = mat->E[g];
    nu[k] = mat->nu[g];
    G[k] = gG[g];
  }
  for (int32_t k = 0; k < P.n_quads; ++k) {
    const int32_t g = L.quad_gid[k];
    for (int b = 0; b < B; ++b) t[(size_t)b * P.n_quads + k] = sec->t[g];
    E[P.n_beams + k] = mat->E[mesh->n_beams + g];
    nu[P.n_beams + k] = mat->nu[mesh->n_beams + g];
    G[P.n_beams + k] = gG[mesh->n_beams + g];
  }
  std::vector<int32_t> own_gid(P.n_own_quads);
  for (int32_t k = 0; k < P.n_own_quads; ++k) own_gid[k] = L.quad_gid[L.own_quad_local[k]];
  std::vector<int32_t> send;
  P.send_off.clear();
  for (const NeighborPlan& nb : L.nbrs) {
    P.send_off.push_back((int64_t)send.size());
    send.insert(send.end(), nb.send_local.begin(), nb.send_local.end());
  }
  P.n_send = (int64_t)send.size();

  int r;
#define UP(dst, src, n) if ((r = upload(h, &P.dst, src, n))) return r
#define AL(dst, n) if ((r = dalloc(h, &P.dst, n))) return r
  UP(x, x.data(), (int64_t)B * P.n_nodes);
  UP(y, y.data(), (int64_t)B * P.n_nodes);
  UP(z, z.data(), (int64_t)B * P.n_nodes);
  UP(beam_conn, L.beam_conn.data(), 2 * (int64_t)P.n_beams);
  UP(quad_conn, L.quad_conn.data(), 4 * (int64_t)P.n_quads);
  UP(A, A.data(), P.n_beams);
  UP(Iy, Iy.data(), P.n_beams);
  UP(Iz, Iz.data(), P.n_beams);
  UP(J, Jt.data(), P.n_beams);
  UP(t, t.data(), (int64_t)B * P.n_quads);
  UP(E, E.data(), ne);
  UP(nu, nu.data(), ne);
  UP(G, G.data(), ne);
  UP(fixed_mask, mask.data(), P.n_nodes);
  if (P.sym) {  // the device works on the upper graph; the full one stays on the host for exports
    UP(node_ptr, P.up.uptr.data(), P.n_nodes + 1);
    UP(node_col, P.up.ucol.data(), P.up.n_ublocks());
    UP(contrib_ptr, P.up.ucontrib_ptr.data(), P.up.n_ublocks() + 1);
    UP(contrib, P.up.ucontrib.data(), (int64_t)P.up.ucontrib.size());
    UP(lptr, P.up.lptr.data(), P.n_nodes + 1);
    UP(lpull, P.up.lpull.data(), (int64_t)P.up.lpull.size());
    std::vector<int32_t> desc;
    build_pull_desc(P.up, desc);
    UP(pdesc, desc.data(), (int64_t)desc.size());
  } else {
    UP(node_ptr, P.pat.node_ptr.data(), P.n_nodes + 1);
    UP(node_col, P.pat.node_col.data(), P.n_blocks);
    UP(contrib_ptr, P.pat.contrib_ptr.data(), P.n_blocks + 1);
    UP(contrib, P.pat.contrib.data(), P.n_staged);
  }
  UP(inc_ptr, P.pat.inc_ptr.data(), P.n_nodes + 1);
  UP(inc_slot, P.pat.inc_slot.data(), P.n_slots);
  if (P.fused) {
    const std::vector<int32_t>& rk = P.sym ? P.up.urank : P.pat.block_rank;
    UP(block_rank, rk.data(), 16 * (int64_t)P.n_quads);
    // per (owned node, incident slot) record {quad, local index, its 4 nodes, its 4 block ranks
    // (int8, -1 = not stored), 0}; quad -1 pads: the fused kernel's load chain node ->
    // incidence -> element -> coordinates becomes record -> coordinates
    P.inc_pad = std::max(4, (P.max_inc + 3) / 4 * 4);
    std::vector<int32_t> rec((size_t)8 * P.n_own * P.inc_pad, 0);
    for (int32_t n = 0; n < P.n_own; ++n) {
      const int64_t i0 = P.pat.inc_ptr[n], ni = P.pat.inc_ptr[n + 1] - i0;
      for (int kk = 0; kk < P.inc_pad; ++kk) {
        int32_t* o = rec.data() + 8 * ((int64_t)n * P.inc_pad + kk);
        if (kk >= ni) {
          o[0] = -1;
          continue;
        }
        const int32_t slot = P.pat.inc_slot[i0 + kk];  // 4 q + il (quad meshes)
        const int64_t q = slot >> 2;
        const int il = slot & 3;
        o[0] = (int32_t)q;
        o[1] = il;
        uint32_t r4 = 0;
        for (int c = 0; c < 4; ++c) {
          o[2 + c] = L.quad_conn[4 * q + c];
          r4 |= (uint32_t)(uint8_t)(int8_t)rk[16 * q + 4 * il + c] << (8 * c);
        }
        o[6] = (int32_t)r4;
      }
    }
    UP(inc_rec, rec.data(), (int64_t)rec.size());
  }
  UP(own_quad_local, L.own_quad_local.data(), P.n_own_quads);
  UP(own_quad_gid, own_gid.data(), P.n_own_quads);
  UP(send_idx, send.data(), P.n_send);
  AL(sendbuf, 6 * std::max<int64_t>(P.n_send, 1));
  AL(stage, B * P.bs.stage);
  AL(vals, B * P.bs.nnz);
  if (P.pull) CK(h, cudaMemset(P.vals, 0, B * P.bs.nnz * sizeof(double)));  // record pads stay zero
  if (P.pull && make_pull_tmap(P.vals, B * P.bs.nnz / PULL_BLOCK, &P.pull_tmap)) {
    h->err = "storage 3: cuTensorMapEncodeTiled failed";
    return SSO_E_CUDA;
  }
  AL(dinv, B * P.ndof);
  if (h->precond == 1) {
    AL(binv, 21 * (int64_t)B * std::max<int32_t>(P.n_own, 1));
    AL(zb, B * P.ndof);
  }
  AL(f, B * P.ndof);
  AL(fbc, B * P.ndof);
  AL(xs, B * P.ndof);
  AL(r, B * P.ndof);
  AL(p, B * P.ndof);
  {
    const char* env = getenv("SSO_CG_FUSED");
    const int fg = h->precond == 1 ? cg_block_fused_grid() : cg_fused_grid();
    P.cgf = B <= fg && L.n_parts == 1 && !h->use_nccl && h->check_every % 2 == 0 &&
            !(env && env[0] == '0');
  }
  if (P.cgf) {
    AL(p2, B * P.ndof);
    CK(h, cudaMemset(P.p2, 0, B * P.ndof * sizeof(double)));
    const char* env = getenv("SSO_SMALL");
    P.small = h->precond == 0 && P.pull && P.n_own == P.n_nodes && cg_small_fits(P.n_own) &&
              !(env && env[0] == '0');
    for (int32_t n = 0; P.small && n < P.n_nodes; ++n)  // every node within the pull descriptor
      P.small = P.up.uptr[n + 1] - P.up.uptr[n] <= 5 && P.up.lptr[n + 1] - P.up.lptr[n] <= 4;
  }
  AL(q, B * P.ndof);
  AL(tmp, B * P.ndof);
  if (L.n_parts > 1 || h->use_nccl) {  // partitioned: single-reduction CG vectors (cg_sr.cu)
    AL(u_sr, B * P.ndof);
    AL(s_sr, B * P.ndof);
    CK(h, cudaMemset(P.u_sr, 0, B * P.ndof * sizeof(double)));
    // rows that read no halo value form the interior range [bnd_lo, bnd_hi): the widest run
    // between owned nodes with a halo neighbour (strips of a grid: every row but the first
    // and last node rows of the strip)
    std::vector<int32_t> bnd;
    for (int32_t n = 0; n < P.n_own; ++n)
      for (int64_t k = P.pat.node_ptr[n]; k < P.pat.node_ptr[n + 1]; ++k)
        if (P.pat.node_col[k] >= P.n_own) {
          bnd.push_back(n);
          break;
        }
    int32_t prev = -1, best = -1;
    bnd.push_back(P.n_own);
    for (int32_t b : bnd) {
      if (b - prev - 1 > best) {
        best = b - prev - 1;
        P.bnd_lo = prev + 1;
        P.bnd_hi = b;
      }
      prev = b;
    }
  }
  AL(gu, B * P.ndof);
  AL(gf, B * P.ndof);
  AL(partial, B * P.bs.partial);
  AL(st, B);
  AL(flags, B);
  AL(tickets, 16);
  AL(scal, 8);
  AL(slot_partial, B * P.bs.slot);
  AL(dxyz, 3 * (int64_t)B * P.n_nodes);
  AL(dt, (int64_t)B * std::max<int32_t>(P.n_quads, 1));
  AL(dt_own, std::max<int32_t>(P.n_own_quads, 1));
  AL(dE, (int64_t)B * std::max<int64_t>(ne, 1));
  // Lanczos history: the first CG segment of up to 2^18 iterations per design (2^20 / B, at least 4096, for
  // batches); longer solves keep the leading 2^18 coefficients (still interlacing Ritz values)
  P.lz_cap = (int)std::min<int64_t>(h->max_iter, B == 1 ? (1 << 18) : std::max(4096, (1 << 20) / B));
  AL(lz_hist, 2 * (int64_t)B * P.lz_cap);
  AL(lz_T, 2 * (int64_t)B * P.lz_cap);
  AL(mscale_d, B);
  P.mscale_h.assign((size_t)B, 0.0);
  P.h_nu = nu;
  P.g_derived.assign((size_t)ne, mat->G ? 0 : 1);
#undef UP
#undef AL
  CK(h, cudaMemset(P.tickets, 0, 16 * sizeof(unsigned)));
  CK(h, cudaMemset(P.st, 0, B * sizeof(CgState)));
  CK(h, cudaMemset(P.xs, 0, B * P.ndof * sizeof(double)));
  CK(h, cudaMemset(P.p, 0, B * P.ndof * sizeof(double)));
  CK(h, cudaMemset(P.gu, 0, B * P.ndof * sizeof(double)));
  CK(h, cudaMemset(P.gf, 0, B * P.ndof * sizeof(double)));
  CK(h, cudaMemset(P.f, 0, B * P.ndof * sizeof(double)));
  P.pat.contrib.clear();  // only needed on the device
  P.pat.contrib.shrink_to_fit();
  P.up.ucontrib.clear();
  P.up.ucontrib.shrink_to_fit();
  P.up.lpull.clear();
  P.up.lpull.shrink_to_fit();
  P.pat.inc_slot.clear();
  P.pat.inc_slot.shrink_to_fit();
  return SSO_OK;
}

// --- user buffers <-> parts ------------------------------------------------
// 6-DOF vectors: the user buffer covers nodes [user_node_begin, +user_nodes);
// every part owns a contiguous global node range inside it.
int vec_in(sso_ctx* h, const double* src, double* Part::*dst) {
  for (auto& pp : h->parts) {
    Part& P = *pp;
    const int64_t off = 6 * (int64_t)(P.lm.own_begin - h->user_node_begin);
    CK(h, cudaMemcpyAsync(P.*dst, src + off, (size_t)P.B * P.ndof_own * sizeof(double), kind_in(h), h->stream));
  }
  return SSO_OK;
}

int vec_out(sso_ctx* h, double* dst, double* Part::*src) {
  if (!dst) return SSO_OK;
  for (auto& pp : h->parts) {
    Part& P = *pp;
    const int64_t off = 6 * (int64_t)(P.lm.own_begin - h->user_node_begin);
    CK(h, cudaMemcpyAsync(dst + off, P.*src, (size_t)P.B * P.ndof_own * sizeof(double), kind_out(h), h->stream));
  }
  return SSO_OK;
}

// Per-node / per-quad design arrays (global): parts take their local entries by global id.
int design_in(sso_ctx* h, const double* src, int64_t n_global, double* Part::*dst, bool quads) {
  if (h->nranks > 1) FAIL(h, SSO_E_INVALID, "sso_set_design is not supported on multi-rank handles");
  if (h->parts.size() == 1) {  // [batch][n_global]
    CK(h, cudaMemcpyAsync(h->P0().*dst, src, (size_t)h->batch * n_global * sizeof(double), kind_in(h),
                          h->stream));
    return SSO_OK;
  }
  std::vector<double> all((size_t)n_global);
  CK(h, cudaMemcpy(all.data(), src, all.size() * sizeof(double),
                   h->mem == SSO_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost));
  for (auto& pp : h->parts) {
    Part& P = *pp;
    const std::vector<int32_t>& gid = quads ? P.lm.quad_gid : P.lm.node_gid;
    std::vector<double> loc(gid.size());
    for (size_t i = 0; i < gid.size(); ++i) loc[i] = all[gid[i]];
    CK(h, cudaMemcpy(P.*dst, loc.data(), loc.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  return SSO_OK;
}

// Per-design scale of the preconditioner for the 2-norm error estimate (lanczos.cu
// mscale_kernel): min over parts / ranks, kept on the host after every assembly.
// The kernels and the copy into the pinned h_mscale are stream-ordered; the host reads the
// values when a solve's certification needs them (mscale_read, after that solve's synchronisation).
int mscale_update(sso_ctx* h) {
  const int B = h->batch;
  for (size_t ip = 0; ip < h->parts.size(); ++ip) {
    Part& P = *h->parts[ip];
    CK(h, cudaMemsetAsync(P.mscale_d, 0xff, B * sizeof(unsigned long long), h->stream));
    {
      long long g0 = g_launches;
      launch_mscale(h->stream, P.n_own, P.dinv, P.binv, P.mscale_d, P.bs);
      h->launches += g_launches - g0;
    }
    if (h->use_nccl)  // positive doubles order like their bit patterns: min of the bits
      CKN(h, nccl().AllReduce(P.mscale_d, P.mscale_d, B, ncclUint64, ncclMin, h->comm, h->stream));
    CK(h, cudaMemcpyAsync(h->h_mscale + ip * B, P.mscale_d, B * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, h->stream));
  }
  h->mscale_pending = true;
  return SSO_OK;
}

// m_min per design (min over the parts) from h_mscale; call after a stream synchronisation
// that follows mscale_update's copy
void mscale_read(sso_ctx* h) {
  if (!h->mscale_pending) return;
  const int B = h->batch;
  std::vector<double> m((size_t)B, 0.0);
  for (size_t ip = 0; ip < h->parts.size(); ++ip)
    for (int bd = 0; bd < B; ++bd) {
      const unsigned long long b = h->h_mscale[ip * B + bd];
      double v;
      std::memcpy(&v, &b, sizeof v);
      if (b == ~0ull) v = 0.0;
      m[bd] = ip == 0 ? v : std::min(m[bd], v);
    }
  for (auto& pp : h->parts) pp->mscale_h = m;
  h->mscale_pending = false;
}

// Error estimates of a finished solve (include/sso.h sso_solve_info): with lambda_min the
// smallest Ritz value of M^-1 K (an upper estimate of the true one), r the true residual,
// rz = r^T M^-1 r, and C = f_bc^T x = |x|_K^2 (CG from x0 = 0):
//   |e|_K / |x|_K <= sqrt(rz / (lambda_min C))                    (energy norm)
//   |e|_2 / |x|_2 <= sqrt(rz) / (lambda_min sqrt(m_min)) / |x|_2   (m_min <= lambda_min(M))
void fill_cert(sso_ctx* h, int bd, const CgState& S, sso_solve_info& info) {
  const double nanv = std::nan("");
  info.lanczos_lmin = S.lz_min;
  info.lanczos_lmax = S.lz_max;
  info.lanczos_iters = S.lz_n;
  const double lmin = S.lz_min, rz = S.red[1], fx = S.red[2], xx = S.red[3];
  mscale_read(h);
  const double mmin = h->P0().mscale_h[bd];
  info.err_energy_est = (lmin > 0.0 && fx > 0.0 && rz >= 0.0) ? std::sqrt(rz / (lmin * fx)) : nanv;
  info.err2_est = (lmin > 0.0 && mmin > 0.0 && xx > 0.0 && rz >= 0.0)
                      ? std::sqrt(rz) / (lmin * std::sqrt(mmin)) / std::sqrt(xx)
                      : nanv;
}

}  // namespace

extern "C" {

int sso_options_default(sso_options* o) {
  if (!o) return SSO_E_INVALID;
  std::memset(o, 0, sizeof(*o));
  o->rtol = 1e-10;
  o->max_iter = 200000;
  o->drill_alpha = 1e-3;
  o->warm_start = 0;
  o->check_every = 64;
  o->mem = SSO_MEM_HOST;
  o->cuda_stream = nullptr;
  o->device = -1;
  o->n_parts = 1;
  o->part_ranges = nullptr;
  o->nranks = 1;
  o->rank = 0;
  o->nccl_unique_id = nullptr;
  o->batch = 1;
  o->reliable = 1;
  o->assembly = 0;
  o->storage = 0;
  o->precond = 0;
  return SSO_OK;
}

const char* sso_last_error(sso_handle h) { return h ? h->err.c_str() : g_create_err.c_str(); }

int sso_nccl_unique_id(void* out) {
  if (!out) return SSO_E_INVALID;
  if (!nccl().ok) {
    g_create_err = nccl().err;
    return SSO_E_NCCL;
  }
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) {
    g_create_err = "ncclGetUniqueId failed";
    return SSO_E_NCCL;
  }
  std::memcpy(out, &id, sizeof(id));
  return SSO_OK;
}

int sso_create(const sso_mesh* mesh, const sso_sections* sec, const sso_materials* mat,
               const sso_supports* sup, const sso_options* opt, sso_handle* out) {
  TRACE("sso_create");
  if (!out) { g_create_err = "null out"; return SSO_E_INVALID; }
  *out = nullptr;
  std::string err;
  int rc = validate(mesh, sec, mat, sup, err);
  if (rc) { g_create_err = err; return rc; }
  sso_options o;
  sso_options_default(&o);
  if (opt) o = *opt;
  if (!(o.rtol > 0.0) || o.max_iter <= 0 || o.check_every <= 0 || !(o.drill_alpha > 0.0)) {
    g_create_err = "options: rtol, max_iter, check_every and drill_alpha must be > 0";
    return SSO_E_INVALID;
  }
  if (o.nranks < 1 || o.rank < 0 || o.rank >= o.nranks || o.n_parts < 1 ||
      (o.nranks > 1 && o.n_parts != o.nranks && o.n_parts != 1) || o.n_parts > mesh->n_nodes ||
      o.nranks > mesh->n_nodes) {
    g_create_err = "options: need 1 <= n_parts <= n_nodes, 0 <= rank < nranks, and n_parts == nranks (or 1) when nranks > 1";
    return SSO_E_INVALID;
  }
  const int32_t n_parts_total = std::max(o.n_parts, o.nranks);
  std::vector<int32_t> ranges = make_ranges(mesh->n_nodes, n_parts_total, o.part_ranges);
  for (int32_t p = 0; p < n_parts_total; ++p)
    if (ranges[p + 1] <= ranges[p] || ranges[0] != 0 || ranges[n_parts_total] != mesh->n_nodes) {
      g_create_err = "options: part_ranges must be strictly increasing from 0 to n_nodes";
      return SSO_E_INVALID;
    }
  if (o.batch < 1 || (o.batch > 1 && (o.n_parts > 1 || o.nranks > 1))) {
    g_create_err = "options: batch >= 1, and batch > 1 needs n_parts == nranks == 1";
    return SSO_E_INVALID;
  }
  if (o.precond < 0 || o.precond > 1) {
    g_create_err = "options: precond must be 0 or 1";
    return SSO_E_INVALID;
  }
  if (o.storage < 0 || o.storage > 3 || o.storage == 2) {
    g_create_err = "options: storage must be 0, 1 or 3";
    return SSO_E_INVALID;
  }
  if (o.nranks > 1 && !o.nccl_unique_id) {
    g_create_err = "options: nranks > 1 needs nccl_unique_id";
    return SSO_E_INVALID;
  }

  sso_ctx* h = new sso_ctx();
  auto bail = [&](int code) {
    g_create_err = h->err;
    free_all(h);
    delete h;
    return code;
  };
  if (o.device >= 0 && cudaSetDevice(o.device) != cudaSuccess) { h->err = "cudaSetDevice failed"; return bail(SSO_E_CUDA); }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { h->err = "no CUDA device"; return bail(SSO_E_CUDA); }
  if (cudaGetDevice(&h->device) != cudaSuccess) { h->err = "no CUDA device"; return bail(SSO_E_CUDA); }
  h->rtol = o.rtol;
  h->max_iter = o.max_iter;
  h->drill_alpha = o.drill_alpha;
  h->warm_start = o.warm_start;
  h->check_every = o.check_every;
  h->mem = o.mem;
  h->nranks = o.nranks;
  h->rank = o.rank;
  {
    const char* e = getenv("SSO_NCCL_SELF");
    h->use_nccl = o.nranks > 1 ||
                  (o.nranks == 1 && o.n_parts == 1 && o.batch == 1 && o.nccl_unique_id && e && e[0] == '1');
  }
  h->batch = o.batch;
  h->reliable = o.reliable;
  h->assembly = o.assembly;
  h->storage = o.storage == 0 ? 3 : o.storage;
  h->precond = o.precond;  // default: upper blocks + pull SpMV (single-strip handles)
  h->g_nodes = mesh->n_nodes;
  h->g_beams = mesh->n_beams;
  h->g_quads = mesh->n_quads;
  if (o.cuda_stream) {
    h->stream = (cudaStream_t)o.cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) { h->err = "stream create failed"; return bail(SSO_E_CUDA); }
    h->own_stream = true;
  }
  if (cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking) != cudaSuccess) { h->err = "stream create failed"; return bail(SSO_E_CUDA); }

  const int64_t ne = (int64_t)mesh->n_beams + mesh->n_quads;
  std::vector<double> gG((size_t)ne);
  for (int64_t e = 0; e < ne; ++e) gG[e] = mat->G ? mat->G[e] : mat->E[e] / (2.0 * (1.0 + mat->nu[e]));
  std::vector<uint8_t> gmask((size_t)mesh->n_nodes, 0);
  for (int32_t k = 0; k < sup->n; ++k) gmask[sup->node[k]] |= (uint8_t)(sup->mask6[k] & 63);

  std::vector<int32_t> mine;
  if (o.nranks > 1) {
    mine.push_back(o.rank);
  } else {
    for (int32_t p = 0; p < n_parts_total; ++p) mine.push_back(p);
  }
  for (int32_t p : mine) {
    auto P = std::make_unique<Part>();
    std::string perr = build_local_mesh(mesh->n_nodes, mesh->n_beams, mesh->beam_conn, mesh->n_quads,
                                        mesh->quad_conn, ranges.data(), n_parts_total, p, P->lm);
    if (!perr.empty()) { h->err = perr; return bail(SSO_E_INVALID); }
    h->parts.push_back(std::move(P));
    const int r = setup_part(h, *h->parts.back(), mesh, sec, mat, gmask, gG);
    if (r) return bail(r);
  }
  if (o.nranks > 1) {
    h->user_node_begin = ranges[o.rank];
    h->user_nodes = ranges[o.rank + 1] - ranges[o.rank];
    h->user_quads = h->P0().n_own_quads;
  } else {
    h->user_node_begin = 0;
    h->user_nodes = mesh->n_nodes;
    h->user_quads = mesh->n_quads;
  }
  if (h->parts.size() > 1) {  // in-process halo fill: one gather launch for all parts
    std::vector<int4> ent;
    for (size_t pi = 0; pi < h->parts.size(); ++pi) {
      const Part& P = *h->parts[pi];
      for (const NeighborPlan& nb : P.lm.nbrs) {
        if (nb.recv_count == 0) continue;
        const Part& Q = *h->parts[nb.part];
        size_t k = 0;
        while (k < Q.lm.nbrs.size() && Q.lm.nbrs[k].part != P.lm.part) ++k;
        if (k == Q.lm.nbrs.size() || (int64_t)Q.lm.nbrs[k].send_local.size() != nb.recv_count) {
          h->err = "halo plan mismatch between parts";
          return bail(SSO_E_STATE);
        }
        for (int64_t i = 0; i < nb.recv_count; ++i)
          ent.push_back(make_int4((int)pi, P.n_own + (int)(nb.recv_offset + i), nb.part,
                                  Q.lm.nbrs[k].send_local[i]));
      }
    }
    h->n_halo_ent = (int)ent.size();
    int r = upload(h, &h->d_halo_ent, ent.data(), (int64_t)ent.size());
    if (r) return bail(r);
    for (int v = 0; v < 5; ++v) {
      std::vector<double*> base;
      for (auto& pp : h->parts) base.push_back(vec_of(*pp, v));
      if ((r = upload(h, &h->d_vbase[v], base.data(), (int64_t)base.size()))) return bail(r);
    }
  }
  if (h->distributed()) {
    // overlap the halo exchange with the interior rows: NCCL ranks with pull storage (the SpMV
    // takes row ranges); in-process parts only on request (SSO_SPLIT=1, for tests)
    const char* env = getenv("SSO_SPLIT");
    bool all_pull = true;
    for (auto& pp : h->parts) all_pull &= pp->pull;
    h->split = all_pull && (env ? env[0] == '1' : h->use_nccl);
    const char* envc = getenv("SSO_PART_STREAMS");
    if (!h->use_nccl && !h->split && !(envc && envc[0] == '0')) {
      h->part_streams.assign(h->parts.size(), nullptr);
      h->part_ev.assign(h->parts.size(), nullptr);
      for (size_t i = 0; i < h->parts.size(); ++i)
        if (cudaStreamCreateWithFlags(&h->part_streams[i], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->part_ev[i], cudaEventDisableTiming) != cudaSuccess) {
          h->err = "stream / event create failed";
          return bail(SSO_E_CUDA);
        }
    }
    // in-process parts with pull storage: one launch per step for all parts (SSO_MULTI=0: per-part
    // launches on per-part streams, for A/B)
    const char* envm = getenv("SSO_MULTI");
    if (!h->use_nccl && !h->split && all_pull && !(envm && envm[0] == '0')) {
      std::vector<PullPart> pp(h->parts.size());
      std::vector<SrPart> sp(h->parts.size());
      for (size_t i = 0; i < h->parts.size(); ++i) {
        Part& P = *h->parts[i];
        std::memset(&pp[i], 0, sizeof(PullPart));
        pp[i].tmap = P.pull_tmap;
        pp[i].pdesc = P.pdesc;
        pp[i].ucol = P.node_col;
        pp[i].lpull = reinterpret_cast<const int2*>(P.lpull);
        pp[i].vals = P.vals;
        pp[i].x = P.u_sr;
        pp[i].y = P.q;
        pp[i].partial = P.partial;
        pp[i].st = P.st;
        pp[i].n_nodes = P.n_own;
        sp[i] = SrPart{P.binv ? nullptr : P.dinv, P.binv, P.xs, P.r, P.u_sr, P.q, P.p, P.s_sr, P.partial, P.st,
                       P.n_own, 0};
        h->max_own = std::max(h->max_own, P.n_own);
      }
      int r = upload(h, &h->d_pull_parts, pp.data(), (int64_t)pp.size());
      if (r || (r = upload(h, &h->d_sr_parts, sp.data(), (int64_t)sp.size()))) return bail(r);
      for (auto ps : h->part_streams)
        if (ps) cudaStreamDestroy(ps);
      for (auto e : h->part_ev)
        if (e) cudaEventDestroy(e);
      h->part_streams.clear();
      h->part_ev.clear();
    }
    if (h->split || !h->part_streams.empty()) {
      if (cudaStreamCreateWithFlags(&h->side_stream, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess) {
        h->err = "stream / event create failed";
        return bail(SSO_E_CUDA);
      }
    }
  }
  {
    std::vector<CgState*> sts;
    for (auto& pp : h->parts) sts.push_back(pp->st);
    int r = upload(h, &h->d_sts, sts.data(), (int64_t)sts.size());
    if (r) return bail(r);
    if ((h->parts.size() > 1 || (h->use_nccl && o.nranks == 1)) &&
        (r = dalloc(h, &h->d_dt_all, std::max<int32_t>(mesh->n_quads, 1))))
      return bail(r);
  }
  if (h->use_nccl) {
    if (!nccl().ok) { h->err = nccl().err; return bail(SSO_E_NCCL); }
    ncclUniqueId id;
    std::memcpy(&id, o.nccl_unique_id, sizeof(id));
    if (nccl().CommInitRank(&h->comm, o.nranks, id, o.rank) != ncclSuccess) { h->err = "ncclCommInitRank failed"; return bail(SSO_E_NCCL); }
  }
  if (cudaMallocHost(&h->h_st, h->batch * sizeof(CgState)) != cudaSuccess ||
      cudaMallocHost(&h->h_chunk, 2 * h->batch * sizeof(CgState)) != cudaSuccess ||
      cudaMallocHost(&h->h_scal, 8 * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&h->h_C, sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&h->h_flags, h->batch * sizeof(DevFlags)) != cudaSuccess ||
      cudaMallocHost(&h->h_mscale, h->parts.size() * h->batch * sizeof(unsigned long long)) != cudaSuccess) {
    h->err = "cudaMallocHost failed";
    return bail(SSO_E_OOM);
  }
  cudaEventCreate(&h->ev_a);
  cudaEventCreate(&h->ev_b);
  cudaEventCreateWithFlags(&h->ev_done[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->ev_done[1], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->ev_order[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->ev_order[1], cudaEventDisableTiming);
  *out = h;
  return SSO_OK;
}

int sso_set_stream(sso_handle h, void* cuda_stream, sso_mem mem) {
  if (!h) return SSO_E_INVALID;
  ENTER(h);
  if (cuda_stream) {
    if (h->own_stream) {
      cudaStreamSynchronize(h->stream);
      cudaStreamDestroy(h->stream);
    }
    h->own_stream = false;
    h->stream = (cudaStream_t)cuda_stream;
    h->order_legacy = false;
  } else {
    h->order_legacy = (mem == SSO_MEM_DEVICE);
  }
  h->mem = mem;
  return SSO_OK;
}

int sso_set_design(sso_handle h, const double* x, const double* y, const double* z, const double* t) {
  ENTER(h);
  TRACE("sso_set_design");
  if (!h) return SSO_E_INVALID;
  int rc;
  if (x && (rc = design_in(h, x, h->g_nodes, &Part::x, false))) return rc;
  if (y && (rc = design_in(h, y, h->g_nodes, &Part::y, false))) return rc;
  if (z && (rc = design_in(h, z, h->g_nodes, &Part::z, false))) return rc;
  if (t && (rc = design_in(h, t, h->g_quads, &Part::t, true))) return rc;
  if (x || y || z)
    for (auto& g : h->fgrid) g.valid = false;
  h->assembled = false;
  h->solved = false;
  return sync(h);
}

static int assemble_pass(sso_ctx* h, bool unconstrained) {
  for (auto& pp : h->parts) {
    Part& P = *pp;
    const uint8_t* mask = unconstrained ? P.free_mask : P.fixed_mask;
    if (P.fused) {
      Scope sc(h, F_ASSEMBLE);
      launch_quad_assemble_fused(h->stream, P.n_own, P.inc_pad, P.node_ptr, P.node_col, P.inc_rec,
                                 P.x, P.y, P.z, P.t, P.E + P.n_beams,
                                 P.nu + P.n_beams, h->drill_alpha, mask, P.vals, P.dinv, P.flags,
                                 P.bs, P.pull ? 1 : 0);
      continue;
    }
    {
      Scope sc(h, F_ELEMENT);
      launch_beam_elements(h->stream, P.n_beams, P.x, P.y, P.z, P.beam_conn, P.A, P.Iy, P.Iz, P.J, P.E,
                           P.G, P.stage, P.flags, P.bs);
      launch_quad_elements(h->stream, P.n_quads, P.x, P.y, P.z, P.quad_conn, P.t, P.E + P.n_beams,
                           P.nu + P.n_beams, h->drill_alpha, P.stage + 36 * 4 * (int64_t)P.n_beams,
                           P.flags, P.bs);
    }
    {
      Scope sc(h, F_ASSEMBLE);
      launch_assemble(h->stream, P.n_own, P.node_ptr, P.node_col, P.contrib_ptr, P.contrib, P.stage,
                      mask, P.vals, P.dinv, P.flags, P.bs, P.pull ? 1 : 0);
    }
  }
  CKL(h);
  return SSO_OK;
}

int sso_assemble(sso_handle h) {
  ENTER(h);
  TRACE("sso_assemble");
  if (!h) return SSO_E_INVALID;
  int rc = reset_flags(h);
  if (rc) return rc;
  if (h->prescribed) {
    // lifting (reading c18): K_full b with the unconstrained matrix, then the real one
    if ((rc = assemble_pass(h, true))) return rc;
    Part& P = h->P0();
    {
      Scope sc(h, F_SPMV);
      spmv_apply(h->stream, P, P.pb, P.kb, nullptr);
    }
    CKL(h);
  }
  if ((rc = assemble_pass(h, false))) return rc;
  if (h->precond == 1) {
    for (auto& pp : h->parts) {
      Part& P = *pp;
      Scope sc(h, F_ASSEMBLE);
      launch_block_inverse(h->stream, P.n_own, P.node_ptr, P.node_col, P.vals, P.pull ? 3 : 0, P.binv,
                           P.flags, P.bs);
    }
    CKL(h);
  }
  // m_min (certification) is enqueued before the flag check: its copy completes under the
  // check's synchronisation
  if ((rc = mscale_update(h))) return rc;
  rc = check_flags(h);
  if (rc) return rc;
  h->assembled = true;
  h->solved = false;
  return SSO_OK;
}

// Reliable update of the residual (SURVEY.md §7 "parity at 1e-9 through CG"):
// r = f_bc - K x for the designs cg_check selects; REPL_FINAL also restarts p = z.
static int replace_step(sso_ctx* h, int mode) {
  int rc;
  long long g0 = g_launches;
  if ((rc = exchange(h, V_X))) return rc;
  for (auto& pp : h->parts) {
    Part& P = *pp;
    spmv_apply(h->stream, P, P.xs, P.tmp, nullptr);
    launch_cg_true_res(h->stream, (int)P.ndof_own, P.fbc, P.tmp, P.partial, P.st, P.bs);
  }
  if ((rc = allreduce(h, 1))) return rc;
  for (auto& pp : h->parts) {
    Part& P = *pp;
    launch_cg_check(h->stream, P.st, mode, P.B);
    if (h->distributed()) {  // single-reduction CG: restart from the true residual (beta = 0 next)
      launch_cgsr_replace(h->stream, P.n_own, P.fbc, P.tmp, P.dinv, P.binv, P.r, P.u_sr, P.partial, P.st);
      continue;
    }
    // fused form: a chunk (even length) ends with the current p in P.p, the previous in
    // P.p2; a replaced r re-forms p from the previous one (the classic form forms p in
    // the next iteration's p update)
    if (P.binv) {
      launch_cg_replace_block(h->stream, P.n_own, P.fbc, P.tmp, P.binv, P.r, P.zb, P.partial, P.st, mode, P.bs);
      if (P.cgf) launch_cg_pfix_z(h->stream, (int)P.ndof_own, P.zb, P.p2, P.p, P.st, P.bs);
    } else {
      launch_cg_replace(h->stream, (int)P.ndof_own, P.fbc, P.tmp, P.dinv, P.r, P.p, P.partial, P.st, mode, P.bs);
      if (P.cgf) launch_cg_pfix(h->stream, (int)P.ndof_own, P.dinv, P.r, P.p2, P.p, P.st, P.bs);
    }
  }
  h->launches += g_launches - g0;
  return SSO_OK;
}

// CG loop as replays of captured chunks of check_every iterations (single part
// and partitioned alike), with reliable residual updates between chunks and a
// final true-residual check that restarts CG when the recurrence has drifted.
static int solve_chunks(sso_ctx* h) {
  Part& P = h->P0();
  int rc;
  const bool prof = h->tm.on;
  if (!h->distributed() && P.small && h->reliable < 2) {
    // small models: the cluster kernel runs to convergence (or max_iter) in ONE launch and the
    // final true-residual check follows in stream order -- one host synchronisation per pass
    // instead of chunk polling
    for (int pass = 0; pass <= MAX_RESTARTS; ++pass) {
      long long g0 = g_launches;
      launch_cg_small(h->stream, P.n_own, (int)std::min<long long>(h->max_iter, INT_MAX), P.pdesc, P.vals, P.dinv,
                      P.xs, P.r, P.p, P.p2, P.st, P.bs);
      h->launches += g_launches - g0;
      if (h->reliable == 0) break;
      if ((rc = replace_step(h, REPL_FINAL))) return rc;
      CK(h, cudaMemcpyAsync(h->h_chunk, P.st, P.B * sizeof(CgState), cudaMemcpyDeviceToHost, h->stream));
      if ((rc = sync(h))) return rc;
      bool restarted = false;
      for (int bd = 0; bd < P.B; ++bd) restarted |= h->h_chunk[bd].done == 0;
      if (!restarted) break;
    }
    return SSO_OK;
  }
  if (!prof && !h->chunk_exec) {
    if ((rc = build_chunk_graph(h, -1, &h->chunk_exec))) return rc;
  }
  if (prof && !h->prof_exec[0]) {
    if ((rc = build_chunk_graph(h, 0, &h->prof_exec[0]))) return rc;
    if ((rc = build_chunk_graph(h, 1, &h->prof_exec[1]))) return rc;
  }
  // Device-side loop in chunks of check_every iterations (graph replays); kernels
  // after convergence return immediately.  One chunk is always queued ahead of the
  // state snapshot being polled, so the GPU never idles on the host.  With
  // profiling on, slot-alternating graphs carry event nodes around every 16th
  // SpMV and the elapsed times of the sampled iterations that ran are accumulated.
  const int64_t max_chunks = (h->max_iter + h->check_every - 1) / h->check_every + 1;
  long long iters_before = 0;
  for (int pass = 0; pass <= MAX_RESTARTS; ++pass) {
    int64_t launched = 0;
    auto launch_chunk = [&](int slot) -> int {
      CK(h, cudaGraphLaunch(prof ? h->prof_exec[slot] : h->chunk_exec, h->stream));
      h->launches += h->kernels_per_chunk;
      CK(h, cudaMemcpyAsync(&h->h_chunk[slot * P.B], P.st, P.B * sizeof(CgState), cudaMemcpyDeviceToHost,
                            h->stream));
      CK(h, cudaEventRecord(h->ev_done[slot], h->stream));
      ++launched;
      return SSO_OK;
    };
    if ((rc = launch_chunk(0))) return rc;
    for (int64_t k = 0;; ++k) {
      const int slot = (int)(k & 1);
      if (launched < max_chunks && (rc = launch_chunk(1 - slot))) return rc;
      CK(h, cudaEventSynchronize(h->ev_done[slot]));
      // batch: the chunk's kernels ran while any design was active
      bool all_done = true, want_repl = false, not_spd = false;
      long long it_max = 0;
      for (int bd = 0; bd < P.B; ++bd) {
        const CgState& Sb = h->h_chunk[slot * P.B + bd];
        all_done &= Sb.done != 0;
        it_max = std::max<long long>(it_max, Sb.iter);
        not_spd |= Sb.done && Sb.status == SSO_E_NOT_SPD;
        want_repl |= !Sb.done && !Sb.floor && Sb.rr < REPL_FACTOR * Sb.rr_ref;
      }
      if (prof) {
        long long ran = it_max - iters_before;
        if (not_spd && ran < h->check_every) ran += 1;
        iters_before = it_max;
        // (the persistent small-model kernel has no per-iteration SpMV to sample)
        for (long long i = 0; !P.small && i < std::min<long long>(ran, h->check_every); i += PROF_EVERY) {
          float ms = 0.f;
          CK(h, cudaEventElapsedTime(&ms, h->chunk_ev[slot][2 * i], h->chunk_ev[slot][2 * i + 1]));
          h->tm.total_ms[F_SPMV] += ms;
          h->tm.launches[F_SPMV] += 1;
        }
      }
      if (all_done || launched == k + 1) break;
      // periodic replacements are a single-part refinement; the partitioned single-reduction CG
      // restarts from the true residual at the end only
      if (h->reliable >= 2 && want_repl && !h->distributed() && (rc = replace_step(h, REPL_PERIODIC))) return rc;
    }
    // converged by the recurrence: check the true residual, restart if it drifted
    if (h->reliable == 0) break;
    if ((rc = replace_step(h, REPL_FINAL))) return rc;
    CK(h, cudaMemcpyAsync(h->h_chunk, P.st, P.B * sizeof(CgState), cudaMemcpyDeviceToHost, h->stream));
    if ((rc = sync(h))) return rc;
    bool restarted = false;
    for (int bd = 0; bd < P.B; ++bd) restarted |= h->h_chunk[bd].done == 0;
    if (!restarted) break;
  }
  return SSO_OK;
}

int sso_solve(sso_handle h, const double* f, double* u, sso_solve_info* info) {
  ENTER(h);
  TRACE("sso_solve");
  const bool add_load = h && h->area_load && !h->skip_load;
  if (!h || (!f && !add_load) || !u) {
    if (h) h->err = "null argument";
    return SSO_E_INVALID;
  }
  if (!h->assembled) FAIL(h, SSO_E_STATE, "sso_solve before sso_assemble");
  int rc;
  const bool dist = h->distributed();
  if (f) {
    if ((rc = vec_in(h, f, &Part::f))) return rc;
  } else {
    for (auto& pp : h->parts)
      CK(h, cudaMemsetAsync(pp->f, 0, (size_t)pp->B * pp->ndof * sizeof(double), h->stream));
  }
  if (add_load) {
    for (auto& pp : h->parts) {
      Part& P = *pp;
      Scope sc(h, F_REDUCE);
      launch_area_load(h->stream, P.n_own, P.n_beams, P.n_quads, P.x, P.y, P.z, P.quad_conn, P.t, P.ld_q, P.ld_w,
                       h->ld_dir, P.inc_ptr, P.inc_slot, P.ld_a, P.f, P.bs);
    }
    CKL(h);
  }
  const int warm = h->warm_start ? 1 : 0;
  if (warm) {
    if ((rc = vec_in(h, u, &Part::xs))) return rc;
    for (auto& pp : h->parts) {
      Scope sc(h, F_UPDATE);
      launch_zero_fixed(h->stream, (int)pp->ndof_own, pp->fixed_mask, pp->xs, pp->bs);
    }
    if ((rc = exchange(h, V_X))) return rc;
    for (auto& pp : h->parts) {
      Part& P = *pp;
      Scope sc(h, F_SPMV);
      spmv_apply(h->stream, P, P.xs, P.tmp, nullptr);
    }
  }
  std::memset(h->h_st, 0, h->batch * sizeof(CgState));
  for (int bd = 0; bd < h->batch; ++bd) {
    h->h_st[bd].tol2 = h->rtol * h->rtol;
    h->h_st[bd].max_iter = h->max_iter;
    h->h_st[bd].dist = dist ? 1 : 0;
    h->h_st[bd].defer_alpha = (!dist && h->P0().cgf) ? 1 : 0;  // the fused update forms alpha
    h->h_st[bd].tol2_rel = h->rtol * h->rtol;
    if (dist) h->h_st[bd].ff = -1.0;  // single-reduction CG: |f_bc|^2 arrives with the first allreduce
  }
  for (auto& pp : h->parts) {
    for (int bd = 0; bd < h->batch; ++bd) {  // this part's Lanczos history
      h->h_st[bd].lz = pp->lz_hist + 2 * (int64_t)bd * pp->lz_cap;
      h->h_st[bd].lz_cap = pp->lz_cap;
    }
    CK(h, cudaMemcpyAsync(pp->st, h->h_st, pp->B * sizeof(CgState), cudaMemcpyHostToDevice, h->stream));
    // the pinned staging struct is reused by the next part: make the upload complete first (the
    // last part's upload is ordered before the solve's own host reads of the state, and the
    // next solve rewrites the struct only after this one has synchronised)
    if (pp != h->parts.back() && (rc = sync(h))) return rc;
  }
  const bool lift = h->prescribed && !h->skip_load;
  if (lift) {  // K_ff u_f = f_f - K_fc b (reading c18)
    Part& P = h->P0();
    Scope sc(h, F_UPDATE);
    launch_lincomb(h->stream, (int64_t)P.B * P.ndof, 1.0, P.f, -1.0, P.kb, P.feff);
  }
  CK(h, cudaEventRecord(h->ev_a, h->stream));
  for (auto& pp : h->parts) {
    Part& P = *pp;
    Scope sc(h, F_UPDATE);
    if (dist)  // single-reduction CG (cg_sr.cu): local gamma, r^T r, |f|^2 travel with the first allreduce
      launch_cgsr_init(h->stream, P.n_own, P.f, P.fixed_mask, P.dinv, P.binv, P.fbc, P.xs, P.r, P.u_sr, P.p,
                       P.s_sr, P.partial, P.st, warm, P.tmp);
    else if (P.binv)
      launch_cg_init_block(h->stream, P.n_own, lift ? P.feff : P.f, P.fixed_mask, P.binv, P.fbc, P.xs, P.r, P.p,
                           P.zb, P.partial, P.st, warm, P.tmp, P.bs);
    else
      launch_cg_init(h->stream, (int)P.ndof_own, lift ? P.feff : P.f, P.fixed_mask, P.dinv, P.fbc, P.xs, P.r,
                     P.p, P.partial, P.st, warm, P.tmp, P.bs);
  }
  {
    TRACE("cg_loop");
    rc = solve_chunks(h);
  }
  if (rc) return rc;
  CK(h, cudaEventRecord(h->ev_b, h->stream));
  // true residual |f_bc - K x| / |f_bc|: local sums of squares into red[0], allreduced
  if ((rc = exchange(h, V_X))) return rc;
  for (auto& pp : h->parts) {
    Part& P = *pp;
    long long g1 = g_launches;
    spmv_apply(h->stream, P, P.xs, P.tmp, nullptr);
    launch_cert_sums(h->stream, P.n_own, P.fbc, P.tmp, P.xs, P.dinv, P.binv, P.partial, P.st, P.bs);
    h->launches += g_launches - g1;
  }
  if ((rc = allreduce(h, 4))) return rc;
  {  // extreme Ritz values of M^-1 K from part 0's coefficient history (the same in every part)
    TRACE("certification");
    Part& P = h->P0();
    long long g1 = g_launches;
    launch_lanczos_ritz(h->stream, P.st, P.lz_T, P.lz_cap, P.B);
    h->launches += g_launches - g1;
  }
  CK(h, cudaMemcpyAsync(h->h_st, h->P0().st, h->batch * sizeof(CgState), cudaMemcpyDeviceToHost,
                        h->stream));
  if (lift) {  // u = u_f + b
    Part& P = h->P0();
    Scope sc(h, F_UPDATE);
    launch_lincomb(h->stream, (int64_t)P.B * P.ndof, 1.0, P.xs, 1.0, P.pb, P.xs);
  }
  if ((rc = vec_out(h, u, &Part::xs))) return rc;
  if ((rc = sync(h))) return rc;
  CKL(h);
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, h->ev_a, h->ev_b) != cudaSuccess) (void)cudaGetLastError();
  int status = SSO_OK, worst = 0;
  for (int bd = 0; bd < h->batch; ++bd) {
    const CgState& Sb = h->h_st[bd];
    const int st_b = Sb.done ? Sb.status : SSO_E_NOT_CONVERGED;
    if (info) {
      info[bd].iters = Sb.iter;
      info[bd].rel_res = Sb.ff > 0 ? std::sqrt(Sb.rr / Sb.ff) : 0.0;
      info[bd].true_rel_res = Sb.ff > 0 ? std::sqrt(Sb.red[0] / Sb.ff) : 0.0;
      fill_cert(h, bd, Sb, info[bd]);
      info[bd].ms = ms;
      info[bd].status = st_b;
    }
    if (st_b == SSO_E_NOT_SPD || (st_b != SSO_OK && status == SSO_OK)) {
      status = st_b;
      worst = bd;
    }
  }
  const CgState& S = h->h_st[worst];
  h->solved = (status == SSO_OK);
  if (status == SSO_E_NOT_SPD) FAIL(h, SSO_E_NOT_SPD, "CG breakdown: p^T K p <= 0 (matrix not SPD)");
  if (status == SSO_E_NOT_CONVERGED) {
    char buf[160];
    snprintf(buf, sizeof buf, "CG not converged after %lld iterations (rel_res %.3e)", S.iter,
             S.ff > 0 ? std::sqrt(S.rr / S.ff) : 0.0);
    h->err = buf;
    h->solved = true;  // u holds the last iterate
    return SSO_E_NOT_CONVERGED;
  }
  return SSO_OK;
}

// Objective + gradient at the parts' (fv, uvec) state (owned entries set; halos exchanged here).
static int grad_impl(sso_ctx* h, sso_objective obj, double* Part::*fv, int uvec, double* C,
                     double* dC_dxyz, double* dC_dt, double* dC_dE = nullptr) {
  const double s = (obj == SSO_OBJ_STRAIN_ENERGY) ? 0.5 : 1.0;
  int rc;
  if ((rc = exchange(h, uvec))) return rc;
  for (auto& pp : h->parts) {
    Part& P = *pp;
    double* U = vec_of(P, uvec);
    {
      Scope sc(h, F_REDUCE);
      launch_dot_local(h->stream, (int)P.ndof_own, P.*fv, U, P.partial, P.st, P.bs);
    }
    {
      Scope sc(h, F_GRAD);
      double* dE = dC_dE ? P.dE : nullptr;
      launch_beam_grad(h->stream, P.n_beams, P.x, P.y, P.z, P.beam_conn, P.A, P.Iy, P.Iz, P.J, P.E, P.G,
                       U, s, P.slot_partial, dE, P.n_beams + P.n_quads, P.bs);
      launch_quad_grad(h->stream, P.n_beams, P.n_quads, P.x, P.y, P.z, P.quad_conn, P.t, P.E, P.nu,
                       h->drill_alpha, U, s, P.slot_partial, P.dt, dE, P.bs);
      // design-dependent load: dC/dp += 2 s u^T df/dp (reading c17)
      if (h->area_load)
        launch_area_load_grad(h->stream, P.n_beams, P.n_quads, P.x, P.y, P.z, P.quad_conn, P.t, P.ld_q, P.ld_w,
                              h->ld_dir, U, 2.0 * s, P.slot_partial, P.dt, P.bs);
    }
    {
      Scope sc(h, F_REDUCE);
      launch_node_reduce(h->stream, P.n_own, P.inc_ptr, P.inc_slot, P.slot_partial, P.dxyz, P.bs);
      if (h->distributed()) launch_gather(h->stream, P.n_own_quads, P.own_quad_local, P.dt, P.dt_own);
    }
  }
  if ((rc = allreduce(h, 1))) return rc;
  CKL(h);
  if (dC_dxyz && h->batch > 1) {
    CK(h, cudaMemcpyAsync(dC_dxyz, h->P0().dxyz, (size_t)h->batch * 3 * h->user_nodes * sizeof(double),
                          kind_out(h), h->stream));
  } else if (dC_dxyz) {
    for (auto& pp : h->parts) {
      Part& P = *pp;
      for (int a = 0; a < 3; ++a)
        CK(h, cudaMemcpyAsync(dC_dxyz + (int64_t)a * h->user_nodes + (P.lm.own_begin - h->user_node_begin),
                              P.dxyz + (int64_t)a * P.n_own, (size_t)P.n_own * sizeof(double), kind_out(h),
                              h->stream));
    }
  }
  if (dC_dE) {
    Part& P = h->P0();
    if (h->simp_chain) launch_simp_chain(h->stream, P.n_beams + P.n_quads, h->batch, P.rho, h->penal, P.E0, P.dE);
    CK(h, cudaMemcpyAsync(dC_dE, P.dE, (size_t)h->batch * (P.n_beams + P.n_quads) * sizeof(double), kind_out(h),
                          h->stream));
  }
  if (dC_dt && h->user_quads > 0) {
    if (!h->distributed()) {
      CK(h, cudaMemcpyAsync(dC_dt, h->P0().dt, (size_t)h->batch * h->user_quads * sizeof(double), kind_out(h),
                            h->stream));
    } else if (h->nranks > 1) {
      CK(h, cudaMemcpyAsync(dC_dt, h->P0().dt_own, (size_t)h->user_quads * sizeof(double), kind_out(h), h->stream));
    } else {
      long long g0 = g_launches;
      for (auto& pp : h->parts) {
        Part& P = *pp;
        launch_scatter(h->stream, P.n_own_quads, P.own_quad_gid, P.dt_own, h->d_dt_all);
      }
      h->launches += g_launches - g0;
      CK(h, cudaMemcpyAsync(dC_dt, h->d_dt_all, (size_t)h->user_quads * sizeof(double), kind_out(h), h->stream));
    }
  }
  CK(h, cudaMemcpyAsync(h->h_st, h->P0().st, h->batch * sizeof(CgState), cudaMemcpyDeviceToHost,
                        h->stream));
  if ((rc = sync(h))) return rc;
  CKL(h);
  if (C) {
    std::vector<double> v(h->batch);
    for (int bd = 0; bd < h->batch; ++bd) v[bd] = s * h->h_st[bd].red[0];
    if (h->mem == SSO_MEM_HOST) {
      std::memcpy(C, v.data(), v.size() * sizeof(double));
    } else {
      CK(h, cudaMemcpy(C, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
  }
  return SSO_OK;
}

static int grad_prescribed(sso_ctx* h, sso_objective obj, double* C, double* dC_dxyz, double* dC_dt,
                           double* dC_dE);

int sso_grad(sso_handle h, sso_objective obj, double* C, double* dC_dxyz, double* dC_dt) {
  ENTER(h);
  TRACE("sso_grad");
  if (!h) return SSO_E_INVALID;
  if (obj != SSO_OBJ_COMPLIANCE && obj != SSO_OBJ_STRAIN_ENERGY) FAIL(h, SSO_E_INVALID, "unknown objective");
  if (!h->solved) FAIL(h, SSO_E_STATE, "sso_grad before a successful sso_solve");
  if (h->prescribed) return grad_prescribed(h, obj, C, dC_dxyz, dC_dt, nullptr);
  return grad_impl(h, obj, &Part::f, V_X, C, dC_dxyz, dC_dt);
}

int sso_grad_at(sso_handle h, sso_objective obj, const double* f, const double* u, double* C,
                double* dC_dxyz, double* dC_dt) {
  ENTER(h);
  TRACE("sso_grad_at");
  if (!h || !f || !u) return SSO_E_INVALID;
  if (obj != SSO_OBJ_COMPLIANCE && obj != SSO_OBJ_STRAIN_ENERGY) FAIL(h, SSO_E_INVALID, "unknown objective");
  if (h->prescribed) FAIL(h, SSO_E_INVALID, "sso_grad_at is not defined with prescribed displacements (use sso_grad)");
  int rc;
  if ((rc = vec_in(h, f, &Part::gf))) return rc;
  if ((rc = vec_in(h, u, &Part::gu))) return rc;
  return grad_impl(h, obj, &Part::gf, V_GU, C, dC_dxyz, dC_dt);
}

// Gradient kernels at state U with scale s into P.dxyz (owned nodes), P.dt, P.dE.
int sso_adjoint_solve(sso_handle h, const double* dg_du, double* lambda, sso_solve_info* info) {
  ENTER(h);
  TRACE("sso_adjoint_solve");
  if (!h || !dg_du || !lambda) return SSO_E_INVALID;
  if (h->distributed()) FAIL(h, SSO_E_INVALID, "sso_adjoint_solve is defined for single-strip handles");
  if (!h->assembled) FAIL(h, SSO_E_STATE, "sso_adjoint_solve before sso_assemble");
  Part& P = h->P0();
  const int64_t nv = (int64_t)P.B * P.ndof;  // every design of a batch
  int r;
  if (!P.ub && (r = dalloc(h, &P.ub, nv))) return r;
  if (!P.fb && (r = dalloc(h, &P.fb, nv))) return r;
  const bool was_solved = h->solved;
  // keep the primal (u, f): the adjoint reuses the CG buffers
  CK(h, cudaMemcpyAsync(P.ub, P.xs, nv * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  CK(h, cudaMemcpyAsync(P.fb, P.f, nv * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  h->skip_load = true;
  const int rc = sso_solve(h, dg_du, lambda, info);  // K symmetric: K^T lambda = K lambda
  h->skip_load = false;
  CK(h, cudaMemcpyAsync(P.xs, P.ub, nv * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  CK(h, cudaMemcpyAsync(P.f, P.fb, nv * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  int rs = sync(h);
  if (rs) return rs;
  h->solved = was_solved;
  return rc;
}

// -lambda^T (dK/dp u - df/dp) [+ s u^T df/dp when u_load_s != 0] at the primal state, lambda in
// P.lam, into P.dxyz / P.dt / P.dE (single strip; every design of a batch, u_load_s only for
// batch 1).  One pass of the bilinear gradient kernels (grad.cu: strains of lambda and u,
// dual numbers through lambda_e^T K_e(p) u_e): PAPER.md Eq. 6 term by term, no polarization.
static int adjoint_grad_dev(sso_ctx* h, double u_load_s) {
  Part& P = h->P0();
  {
    Scope sc(h, F_GRAD);
    launch_beam_grad(h->stream, P.n_beams, P.x, P.y, P.z, P.beam_conn, P.A, P.Iy, P.Iz, P.J, P.E, P.G, P.xs, 1.0,
                     P.slot_partial, P.dE, P.n_beams + P.n_quads, P.bs, P.lam);
    launch_quad_grad(h->stream, P.n_beams, P.n_quads, P.x, P.y, P.z, P.quad_conn, P.t, P.E, P.nu, h->drill_alpha,
                     P.xs, 1.0, P.slot_partial, P.dt, P.dE, P.bs, P.lam);
    // + lambda^T df/dp (design-dependent area loads, reading c17)
    if (h->area_load)
      launch_area_load_grad(h->stream, P.n_beams, P.n_quads, P.x, P.y, P.z, P.quad_conn, P.t, P.ld_q, P.ld_w,
                            h->ld_dir, P.lam, 1.0, P.slot_partial, P.dt, P.bs);
    if (h->area_load && u_load_s != 0.0)
      launch_area_load_grad(h->stream, P.n_beams, P.n_quads, P.x, P.y, P.z, P.quad_conn, P.t, P.ld_q, P.ld_w,
                            h->ld_dir, P.xs, u_load_s, P.slot_partial, P.dt, P.bs);
    launch_node_reduce(h->stream, P.n_own, P.inc_ptr, P.inc_slot, P.slot_partial, P.dxyz, P.bs);
  }
  CKL(h);
  return SSO_OK;
}

int sso_grad_adjoint(sso_handle h, const double* lambda, double* dg_dxyz, double* dg_dt, double* dg_dE) {
  ENTER(h);
  TRACE("sso_grad_adjoint");
  if (!h || !lambda) return SSO_E_INVALID;
  if (h->distributed()) FAIL(h, SSO_E_INVALID, "sso_grad_adjoint is defined for single-strip handles");
  if (!h->solved) FAIL(h, SSO_E_STATE, "sso_grad_adjoint before a successful sso_solve");
  Part& P = h->P0();
  const int64_t ne = (int64_t)P.n_beams + P.n_quads;
  const size_t B = (size_t)P.B;
  int r;
  if (!P.lam && (r = dalloc(h, &P.lam, (int64_t)B * P.ndof))) return r;
  if ((r = vec_in(h, lambda, &Part::lam))) return r;
  if ((r = adjoint_grad_dev(h, 0.0))) return r;
  if (dg_dxyz)
    CK(h, cudaMemcpyAsync(dg_dxyz, P.dxyz, 3 * B * P.n_nodes * sizeof(double), kind_out(h), h->stream));
  if (dg_dt && P.n_quads)
    CK(h, cudaMemcpyAsync(dg_dt, P.dt, B * P.n_quads * sizeof(double), kind_out(h), h->stream));
  if (dg_dE) CK(h, cudaMemcpyAsync(dg_dE, P.dE, B * ne * sizeof(double), kind_out(h), h->stream));
  return sync(h);
}

// Compliance gradient with prescribed displacements (reading c18): C = s f^T u,
// lambda = s u_hom (the same loads with b = 0, one more PCG solve),
// dC/dp = -lambda^T dK/dp u + (lambda + s u)^T df/dp.
static int grad_prescribed(sso_ctx* h, sso_objective obj, double* C, double* dC_dxyz, double* dC_dt,
                           double* dC_dE) {
  const double s = (obj == SSO_OBJ_STRAIN_ENERGY) ? 0.5 : 1.0;
  Part& P = h->P0();
  const int64_t ne = (int64_t)P.n_beams + P.n_quads;
  const int B = P.B;
  const int64_t nv = (int64_t)B * P.ndof;
  if (B > 1 && h->area_load)
    FAIL(h, SSO_E_INVALID, "prescribed displacements with area loads are defined for batch-1 handles");
  int r;
  if (!P.lam && (r = dalloc(h, &P.lam, nv))) return r;
  if (!P.gf && (r = dalloc(h, &P.gf, nv))) return r;
  CK(h, cudaMemcpyAsync(P.gf, P.f, nv * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  // the adjoint solve through the public entry, with device pointers for the call
  const sso_mem mem = h->mem;
  h->mem = SSO_MEM_DEVICE;
  r = sso_adjoint_solve(h, P.gf, P.lam, nullptr);
  h->mem = mem;
  if (r) return r;
  {
    Scope sc(h, F_UPDATE);
    launch_lincomb(h->stream, nv, s, P.lam, 0.0, P.lam, P.lam);
  }
  if ((r = adjoint_grad_dev(h, s))) return r;
  {
    Scope sc(h, F_REDUCE);
    launch_dot_local(h->stream, (int)P.ndof, P.f, P.xs, P.partial, P.st, P.bs);
    CK(h, cudaMemcpyAsync(h->h_chunk, P.st, B * sizeof(CgState), cudaMemcpyDeviceToHost, h->stream));
  }
  if (dC_dxyz)
    CK(h, cudaMemcpyAsync(dC_dxyz, P.dxyz, 3 * (size_t)B * P.n_nodes * sizeof(double), kind_out(h), h->stream));
  if (dC_dt && P.n_quads)
    CK(h, cudaMemcpyAsync(dC_dt, P.dt, (size_t)B * P.n_quads * sizeof(double), kind_out(h), h->stream));
  if (dC_dE) {
    if (h->simp_chain) launch_simp_chain(h->stream, (int)ne, B, P.rho, h->penal, P.E0, P.dE);
    CK(h, cudaMemcpyAsync(dC_dE, P.dE, (size_t)B * ne * sizeof(double), kind_out(h), h->stream));
  }
  if ((r = sync(h))) return r;
  if (C) {
    std::vector<double> v(B);
    for (int d = 0; d < B; ++d) v[d] = s * h->h_chunk[d].red[0];
    if (h->mem == SSO_MEM_HOST) std::memcpy(C, v.data(), B * sizeof(double));
    else CK(h, cudaMemcpy(C, v.data(), B * sizeof(double), cudaMemcpyHostToDevice));
  }
  return SSO_OK;
}

int sso_grad_E(sso_handle h, sso_objective obj, double* dC_dE) {
  ENTER(h);
  TRACE("sso_grad_E");
  if (!h || !dC_dE) return SSO_E_INVALID;
  if (obj != SSO_OBJ_COMPLIANCE && obj != SSO_OBJ_STRAIN_ENERGY) FAIL(h, SSO_E_INVALID, "unknown objective");
  if (h->distributed()) FAIL(h, SSO_E_INVALID, "sso_grad_E is defined for single-strip handles");
  if (!h->solved) FAIL(h, SSO_E_STATE, "sso_grad_E before a successful sso_solve");
  if (h->prescribed) return grad_prescribed(h, obj, nullptr, nullptr, nullptr, dC_dE);
  return grad_impl(h, obj, &Part::f, V_X, nullptr, nullptr, nullptr, dC_dE);
}

int sso_set_prescribed(sso_handle h, const double* b) {
  ENTER(h);
  TRACE("sso_set_prescribed");
  if (!h) return SSO_E_INVALID;
  if (!b) {
    if (h->prescribed) h->assembled = false;
    h->prescribed = false;
    h->solved = false;
    return SSO_OK;
  }
  if (h->distributed()) FAIL(h, SSO_E_INVALID, "sso_set_prescribed is defined for single-strip handles");
  Part& P = h->P0();
  const int64_t nv = (int64_t)P.B * P.ndof;  // one b per design of a batch
  int r;
  if (!P.pb && (r = dalloc(h, &P.pb, nv))) return r;
  if (!P.kb && (r = dalloc(h, &P.kb, nv))) return r;
  if (!P.feff && (r = dalloc(h, &P.feff, nv))) return r;
  if (!P.free_mask) {  // per-node support bitmasks, all clear
    if ((r = dalloc(h, &P.free_mask, P.n_nodes))) return r;
    CK(h, cudaMemsetAsync(P.free_mask, 0, P.n_nodes, h->stream));
  }
  std::vector<double> hb(nv);
  CK(h, cudaMemcpy(hb.data(), b, nv * sizeof(double),
                   h->mem == SSO_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost));
  std::vector<uint8_t> mask(P.n_nodes);
  CK(h, cudaMemcpy(mask.data(), P.fixed_mask, P.n_nodes, cudaMemcpyDeviceToHost));
  for (int64_t k = 0; k < nv; ++k) {
    const int64_t i = k % P.ndof;
    if (!std::isfinite(hb[k])) FAIL(h, SSO_E_INVALID, "sso_set_prescribed: non-finite value");
    if (!((mask[i / 6] >> (i % 6)) & 1)) hb[k] = 0.0;  // only the constrained DOFs carry b
  }
  CK(h, cudaMemcpy(P.pb, hb.data(), nv * sizeof(double), cudaMemcpyHostToDevice));
  h->prescribed = true;
  h->assembled = false;  // K_full b is formed by the next sso_assemble
  h->solved = false;
  return SSO_OK;
}

int sso_set_area_load(sso_handle h, const double* q, const double* w, const double* dir) {
  ENTER(h);
  TRACE("sso_set_area_load");
  if (!h) return SSO_E_INVALID;
  if (!q && !w) {
    h->area_load = false;
    h->solved = false;
    return SSO_OK;
  }
  if (!dir) FAIL(h, SSO_E_INVALID, "sso_set_area_load: dir is NULL");
  for (int a = 0; a < 3; ++a)
    if (!std::isfinite(dir[a])) FAIL(h, SSO_E_INVALID, "sso_set_area_load: non-finite direction");
  const int64_t nq = h->g_quads;
  std::vector<double> hq(nq, 0.0), hw(nq, 0.0);
  const cudaMemcpyKind kh = h->mem == SSO_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost;
  if (nq > 0 && q) CK(h, cudaMemcpy(hq.data(), q, nq * sizeof(double), kh));
  if (nq > 0 && w) CK(h, cudaMemcpy(hw.data(), w, nq * sizeof(double), kh));
  for (int64_t e = 0; e < nq; ++e)
    if (!std::isfinite(hq[e]) || !std::isfinite(hw[e])) FAIL(h, SSO_E_INVALID, "sso_set_area_load: non-finite load");
  int r;
  for (auto& pp : h->parts) {
    Part& P = *pp;
    const int64_t nl = std::max<int64_t>(P.n_quads, 1);
    if (!P.ld_q && (r = dalloc(h, &P.ld_q, nl))) return r;
    if (!P.ld_w && (r = dalloc(h, &P.ld_w, nl))) return r;
    if (!P.ld_a && (r = dalloc(h, &P.ld_a, (int64_t)P.B * nl))) return r;
    std::vector<double> lq(P.n_quads), lw(P.n_quads);
    for (int32_t k = 0; k < P.n_quads; ++k) {
      const int32_t g = P.lm.quad_gid.empty() ? k : P.lm.quad_gid[k];
      lq[k] = hq[g], lw[k] = hw[g];
    }
    if (P.n_quads > 0) {
      CK(h, cudaMemcpy(P.ld_q, lq.data(), P.n_quads * sizeof(double), cudaMemcpyHostToDevice));
      CK(h, cudaMemcpy(P.ld_w, lw.data(), P.n_quads * sizeof(double), cudaMemcpyHostToDevice));
    }
  }
  for (int a = 0; a < 3; ++a) h->ld_dir[a] = dir[a];
  h->area_load = true;
  h->solved = false;
  return SSO_OK;
}

int sso_set_density(sso_handle h, const double* rho, double penal, const double* E0, const double* G0) {
  ENTER(h);
  TRACE("sso_set_density");
  if (!h || !rho || !E0) return SSO_E_INVALID;
  if (h->distributed()) FAIL(h, SSO_E_INVALID, "sso_set_density is defined for single-strip handles");
  if (!(penal >= 1.0) || !std::isfinite(penal)) FAIL(h, SSO_E_INVALID, "sso_set_density: penalty P must be >= 1");
  Part& P = h->P0();
  const int64_t ne = (int64_t)P.n_beams + P.n_quads;
  if (ne == 0) FAIL(h, SSO_E_INVALID, "sso_set_density: no elements");
  const cudaMemcpyKind kin = h->mem == SSO_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost;
  std::vector<double> r((size_t)ne), e0((size_t)ne), g0(G0 ? (size_t)ne : 0);
  CK(h, cudaMemcpy(r.data(), rho, ne * sizeof(double), kin));
  CK(h, cudaMemcpy(e0.data(), E0, ne * sizeof(double), kin));
  if (G0) CK(h, cudaMemcpy(g0.data(), G0, ne * sizeof(double), kin));
  for (int64_t k = 0; k < ne; ++k) {
    if (!(r[k] > 0.0 && r[k] <= 1.0) || !(e0[k] > 0.0) || !std::isfinite(e0[k]) ||
        (G0 && (!(g0[k] > 0.0) || !std::isfinite(g0[k])))) {
      char buf[112];
      snprintf(buf, sizeof buf, "element %lld: rho outside (0, 1] or E0 / G0 <= 0 or non-finite", (long long)k);
      FAIL(h, SSO_E_INVALID, buf);
    }
  }
  int rc;
  if (!P.rho && (rc = dalloc(h, &P.rho, ne))) return rc;
  if (!P.E0 && (rc = dalloc(h, &P.E0, ne))) return rc;
  if (G0 && !P.G0 && (rc = dalloc(h, &P.G0, ne))) return rc;
  CK(h, cudaMemcpy(P.rho, r.data(), ne * sizeof(double), cudaMemcpyHostToDevice));
  CK(h, cudaMemcpy(P.E0, e0.data(), ne * sizeof(double), cudaMemcpyHostToDevice));
  if (G0) CK(h, cudaMemcpy(P.G0, g0.data(), ne * sizeof(double), cudaMemcpyHostToDevice));
  launch_simp_material(h->stream, (int)ne, P.rho, penal, P.E0, G0 ? P.G0 : nullptr, P.nu, P.E, P.G);
  CKL(h);
  // later sso_set_material calls scale G from these moduli
  std::fill(P.g_derived.begin(), P.g_derived.end(), G0 ? 0 : 1);
  h->simp = true;
  h->penal = penal;
  h->assembled = false;
  h->solved = false;
  return sync(h);
}

int sso_grad_density(sso_handle h, sso_objective obj, double* dC_drho) {
  ENTER(h);
  TRACE("sso_grad_density");
  if (!h || !dC_drho) return SSO_E_INVALID;
  if (!h->simp) FAIL(h, SSO_E_STATE, "sso_grad_density without sso_set_density");
  h->simp_chain = true;
  const int rc = sso_grad_E(h, obj, dC_drho);
  h->simp_chain = false;
  return rc;
}

int sso_set_material(sso_handle h, const double* E) {
  ENTER(h);
  TRACE("sso_set_material");
  if (!h || !E) return SSO_E_INVALID;
  if (h->distributed()) FAIL(h, SSO_E_INVALID, "sso_set_material is defined for single-strip handles");
  h->simp = false;
  Part& P = h->P0();
  const int64_t ne = (int64_t)P.n_beams + P.n_quads;
  std::vector<double> e((size_t)ne), g((size_t)ne);
  CK(h, cudaMemcpy(e.data(), E, ne * sizeof(double),
                   h->mem == SSO_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost));
  CK(h, cudaMemcpy(g.data(), P.G, ne * sizeof(double), cudaMemcpyDeviceToHost));
  std::vector<double> eold((size_t)ne);
  CK(h, cudaMemcpy(eold.data(), P.E, ne * sizeof(double), cudaMemcpyDeviceToHost));
  for (int64_t k = 0; k < ne; ++k) {
    if (!(e[k] > 0.0) || !std::isfinite(e[k])) {
      char buf[96];
      snprintf(buf, sizeof buf, "element %lld: E <= 0 or non-finite", (long long)k);
      FAIL(h, SSO_E_INVALID, buf);
    }
    // the whole elastic tensor scales with E (SIMP): a derived G follows E, a given G scales
    g[k] = P.g_derived[k] ? e[k] / (2.0 * (1.0 + P.h_nu[k])) : g[k] * (e[k] / eold[k]);
  }
  CK(h, cudaMemcpy(P.E, e.data(), ne * sizeof(double), cudaMemcpyHostToDevice));
  CK(h, cudaMemcpy(P.G, g.data(), ne * sizeof(double), cudaMemcpyHostToDevice));
  h->assembled = false;
  h->solved = false;
  return SSO_OK;
}

}  // extern "C"

namespace {

// Hat filter (filter.cu).  The cell grid is built here on the host from the current
// design-0 coordinates: cubic cells of edge >= radius, so every point within the
// radius lies in the 27 cells around a point's own cell.
// design bd's coordinates into grid g (the cached grid of design 0, or a per-call grid of a
// batch design)
int build_filter_grid(sso_ctx* h, int on_elements, double radius, int bd, sso_ctx::FilterGrid& g) {
  if (g.valid && g.radius == radius) return SSO_OK;
  free_filter_grid(g);
  Part& P = h->P0();
  const int64_t nn = P.n_nodes;
  const int64_t off = (int64_t)bd * P.bs.node;
  std::vector<double> X(nn), Y(nn), Z(nn);
  CK(h, cudaMemcpyAsync(X.data(), P.x + off, nn * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaMemcpyAsync(Y.data(), P.y + off, nn * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaMemcpyAsync(Z.data(), P.z + off, nn * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  std::vector<double> px, py, pz;
  if (!on_elements) {
    px = X, py = Y, pz = Z;
  } else {  // element centroids, beams then quads (mean of the element's nodes)
    auto add = [&](const std::vector<int32_t>& conn, int k) {
      for (size_t e = 0; e < conn.size() / k; ++e) {
        double a = 0, b = 0, c = 0;
        for (int j = 0; j < k; ++j) {
          const int32_t n = conn[e * k + j];
          a += X[n], b += Y[n], c += Z[n];
        }
        px.push_back(a / k), py.push_back(b / k), pz.push_back(c / k);
      }
    };
    add(P.lm.beam_conn, 2);
    add(P.lm.quad_conn, 4);
  }
  const int64_t n = (int64_t)px.size();
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < n; ++i) {
    const double v[3] = {px[i], py[i], pz[i]};
    for (int a = 0; a < 3; ++a) lo[a] = std::min(lo[a], v[a]), hi[a] = std::max(hi[a], v[a]);
  }
  double cell = radius;
  int64_t dims[3];
  const int64_t max_cells = std::max<int64_t>(8 * n, 1 << 16);
  for (;;) {
    for (int a = 0; a < 3; ++a) dims[a] = (n ? (int64_t)std::floor((hi[a] - lo[a]) / cell) : 0) + 1;
    if (dims[0] * dims[1] * dims[2] <= max_cells) break;
    cell *= 1.5;  // larger cells stay correct (edge >= radius), only less selective
  }
  const int64_t ncell = dims[0] * dims[1] * dims[2];
  std::vector<int32_t> cid(n), cell_of(2 * n), perm(n);
  std::vector<int64_t> start(ncell + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    int64_t c3[3];
    const double v[3] = {px[i], py[i], pz[i]};
    for (int a = 0; a < 3; ++a)
      c3[a] = std::min<int64_t>(dims[a] - 1, (int64_t)std::floor((v[a] - lo[a]) / cell));
    cid[i] = (int32_t)((c3[2] * dims[1] + c3[1]) * dims[0] + c3[0]);
    ++start[cid[i] + 1];
  }
  for (int64_t c = 0; c < ncell; ++c) start[c + 1] += start[c];
  std::vector<int64_t> fill(start.begin(), start.end() - 1);
  std::vector<double> sx(n), sy(n), sz(n);
  for (int64_t i = 0; i < n; ++i) {  // stable: ascending original index within a cell
    const int64_t k = fill[cid[i]]++;
    perm[k] = (int32_t)i;
    cell_of[i] = (int32_t)k;
    cell_of[n + i] = cid[i];
    sx[k] = px[i], sy[k] = py[i], sz[k] = pz[i];
  }
  int rc;
  if ((rc = upload(h, &g.px, sx.data(), n)) || (rc = upload(h, &g.py, sy.data(), n)) ||
      (rc = upload(h, &g.pz, sz.data(), n)) || (rc = upload(h, &g.cell_of, cell_of.data(), 2 * n)) ||
      (rc = upload(h, &g.perm, perm.data(), n)) || (rc = upload(h, &g.cell_start, start.data(), ncell + 1)) ||
      (rc = dalloc(h, &g.io, 6 * n))) {
    free_filter_grid(g);
    return rc;
  }
  g.n = (int32_t)n;
  g.gx = (int)dims[0], g.gy = (int)dims[1], g.gz = (int)dims[2];
  g.radius = radius;
  g.valid = true;
  return SSO_OK;
}

}  // namespace

extern "C" {

int sso_hat_filter(sso_handle h, int32_t on_elements, double radius, int32_t ncomp, const double* in,
                   double* out) {
  ENTER(h);
  TRACE("sso_hat_filter");
  if (!h || !in || !out) return SSO_E_INVALID;
  if (h->distributed()) FAIL(h, SSO_E_INVALID, "sso_hat_filter is defined for single-strip handles");
  if (!(radius > 0.0) || !std::isfinite(radius)) FAIL(h, SSO_E_INVALID, "radius must be positive and finite");
  if (ncomp < 1 || ncomp > 3) FAIL(h, SSO_E_INVALID, "ncomp must be 1, 2 or 3");
  // batch 1: the grid is cached per (kind, radius); a batch builds each design's grid from its
  // own coordinates for this call (in / out [batch][ncomp][n])
  for (int bd = 0; bd < h->batch; ++bd) {
    sso_ctx::FilterGrid tmp;
    sso_ctx::FilterGrid& g = h->batch == 1 ? h->fgrid[on_elements ? 1 : 0] : tmp;
    int rc = build_filter_grid(h, on_elements != 0, radius, bd, g);
    if (rc) return rc;
    const int64_t n = g.n;
    if (n == 0) {
      if (&g == &tmp) free_filter_grid(tmp);
      return SSO_OK;
    }
    const double* din = in + (int64_t)bd * ncomp * n;
    double* dout = out + (int64_t)bd * ncomp * n;
    if (h->mem == SSO_MEM_HOST) {
      CK(h, cudaMemcpyAsync(g.io, din, ncomp * n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
      din = g.io;
      dout = g.io + 3 * n;
    }
    const long long g0 = g_launches;
    launch_hat_filter(h->stream, (int)n, ncomp, g.px, g.py, g.pz, g.cell_of, g.perm, g.cell_start, g.gx, g.gy,
                      g.gz, radius, din, dout);
    CKL(h);
    h->launches += g_launches - g0;
    if (h->mem == SSO_MEM_HOST)
      CK(h, cudaMemcpyAsync(out + (int64_t)bd * ncomp * n, dout, ncomp * n * sizeof(double), cudaMemcpyDeviceToHost,
                            h->stream));
    if ((rc = sync(h))) return rc;
    if (&g == &tmp) free_filter_grid(tmp);
  }
  return SSO_OK;
}

int sso_spmv(sso_handle h, const double* xin, double* yout) {
  ENTER(h);
  TRACE("sso_spmv");
  if (!h || !xin || !yout) return SSO_E_INVALID;
  if (!h->assembled) FAIL(h, SSO_E_STATE, "sso_spmv before sso_assemble");
  int rc;
  if ((rc = vec_in(h, xin, &Part::gu))) return rc;
  if ((rc = exchange(h, V_GU))) return rc;
  for (auto& pp : h->parts) {
    Part& P = *pp;
    Scope sc(h, F_SPMV);
    spmv_apply(h->stream, P, P.gu, P.tmp, nullptr);
  }
  CKL(h);
  if ((rc = vec_out(h, yout, &Part::tmp))) return rc;
  return sync(h);
}

int sso_sizes(sso_handle h, int64_t* ndof, int64_t* nnz, int64_t* n_blocks) {
  if (!h) return SSO_E_INVALID;
  int64_t d = 0, z = 0, b = 0;
  for (auto& pp : h->parts) {
    d += pp->ndof_own;
    z += pp->nnz;
    b += pp->pat.node_ptr[pp->n_own];
  }
  if (ndof) *ndof = d;
  if (nnz) *nnz = z;
  if (n_blocks) *n_blocks = b;
  return SSO_OK;
}

int sso_storage_info(sso_handle h, int64_t* stored_values, int64_t* stored_blocks, int32_t* symmetric) {
  ENTER(h);
  if (!h) return SSO_E_INVALID;
  int64_t v = 0, b = 0;
  bool sym = true, pull = true;
  for (auto& pp : h->parts) {
    v += 36 * pp->stored_blocks;
    b += pp->stored_blocks;
    sym &= pp->sym;
    pull &= pp->pull;
  }
  if (stored_values) *stored_values = v;
  if (stored_blocks) *stored_blocks = b;
  if (symmetric) *symmetric = (sym && pull) ? 3 : 0;
  return SSO_OK;
}


int sso_part_info(sso_handle h, int32_t* n_parts_here, int32_t* own_node_begin, int32_t* own_nodes,
                  int32_t* own_quads) {
  ENTER(h);
  if (!h) return SSO_E_INVALID;
  if (n_parts_here) *n_parts_here = (int32_t)h->parts.size();
  if (own_node_begin) *own_node_begin = h->user_node_begin;
  if (own_nodes) *own_nodes = h->user_nodes;
  if (own_quads) *own_quads = h->user_quads;
  return SSO_OK;
}

int sso_export_csr(sso_handle h, int64_t* row_ptr, int32_t* col_idx, double* vals) {
  ENTER(h);
  if (!h) return SSO_E_INVALID;
  if (vals && !h->assembled) FAIL(h, SSO_E_STATE, "export of values before sso_assemble");
  // rows of the owned nodes of every part, in global node order, columns in
  // ascending GLOBAL order (the local halo numbering permuted back)
  int64_t base = 0, row = 0;
  std::vector<double> pv;
  std::vector<std::pair<int32_t, int32_t>> cols;
  for (auto& pp : h->parts) {
    Part& P = *pp;
    const HostPattern& T = P.pat;
    if (vals) {
      pv.resize((size_t)((P.pull ? PULL_BLOCK : 36) * P.stored_blocks));
      CK(h, cudaMemcpy(pv.data(), P.vals, pv.size() * sizeof(double), cudaMemcpyDeviceToHost));
    }
    // value (a, b) of block (n, k-th full neighbour): symmetric storage keeps the
    // blocks (n, m >= n); a lower block is the transpose of the stored (m, n)
    auto value = [&](int32_t n, int64_t k, int a, int b) -> double {
      const int64_t b0 = T.node_ptr[n];
      const int64_t deg = T.node_ptr[n + 1] - b0;
      if (!P.sym) return pv[36 * b0 + 6 * a * deg + 6 * k + b];
      const int32_t m = T.node_col[b0 + k];
      const UpperPattern& U = P.up;
      // position of (row a, column b) of upper block ku: one PULL_BLOCK record per block (rec_off)
      auto at = [&](int64_t u0, int64_t ud, int64_t ku, int ra, int cb) {
        (void)ud;
        return PULL_BLOCK * (u0 + ku) + rec_off(ra, cb);
      };
      if (m >= n) {
        const int64_t ud = U.uptr[n + 1] - U.uptr[n];
        const int64_t ku = k - (deg - ud);
        return pv[at(U.uptr[n], ud, ku, a, b)];
      }
      const int64_t ud = U.uptr[m + 1] - U.uptr[m];
      const int32_t* c0 = U.ucol.data() + U.uptr[m];
      const int64_t ku = std::lower_bound(c0, c0 + ud, n) - c0;
      return pv[at(U.uptr[m], ud, ku, b, a)];
    };
    for (int32_t n = 0; n < P.n_own; ++n) {
      const int64_t b0 = T.node_ptr[n];
      const int64_t deg = T.node_ptr[n + 1] - b0;
      cols.clear();
      for (int64_t k = 0; k < deg; ++k) cols.push_back({P.lm.node_gid[T.node_col[b0 + k]], (int32_t)k});
      std::sort(cols.begin(), cols.end());
      for (int a = 0; a < 6; ++a) {
        const int64_t start = base + 36 * b0 + 6 * a * deg;
        if (row_ptr) row_ptr[row + a] = start;
        for (int64_t kk = 0; kk < deg; ++kk) {
          const int32_t gcol = cols[kk].first, k = cols[kk].second;
          for (int b = 0; b < 6; ++b) {
            if (col_idx) col_idx[start + 6 * kk + b] = 6 * gcol + b;
            if (vals) vals[start + 6 * kk + b] = value(n, k, a, b);
          }
        }
      }
      row += 6;
    }
    base += P.nnz;
  }
  if (row_ptr) row_ptr[row] = base;
  return SSO_OK;
}

int sso_export_scatter(sso_handle h, int32_t* block_rank) {
  ENTER(h);
  if (!h || !block_rank) return SSO_E_INVALID;
  if (h->distributed()) FAIL(h, SSO_E_INVALID, "sso_export_scatter is defined for single-part handles");
  std::memcpy(block_rank, h->P0().pat.block_rank.data(), h->P0().pat.block_rank.size() * sizeof(int32_t));
  return SSO_OK;
}

int sso_export_ke(sso_handle h, int64_t first, int64_t count, double* ke) {
  ENTER(h);
  if (!h || !ke) return SSO_E_INVALID;
  if (h->distributed()) FAIL(h, SSO_E_INVALID, "sso_export_ke is defined for single-part handles");
  Part& P = h->P0();
  const int64_t ne = (int64_t)P.n_beams + P.n_quads;
  if (first < 0 || count < 0 || first + count > ne) FAIL(h, SSO_E_INVALID, "element range out of bounds");
  if (!h->assembled) FAIL(h, SSO_E_STATE, "export of K_e before sso_assemble");
  // the fused path keeps no element matrices: form them (debug export only)
  launch_beam_elements(h->stream, P.n_beams, P.x, P.y, P.z, P.beam_conn, P.A, P.Iy, P.Iz, P.J, P.E, P.G,
                       P.stage, P.flags, P.bs);
  launch_quad_elements(h->stream, P.n_quads, P.x, P.y, P.z, P.quad_conn, P.t, P.E + P.n_beams,
                       P.nu + P.n_beams, h->drill_alpha, P.stage + 36 * 4 * (int64_t)P.n_beams, P.flags, P.bs);
  CKL(h);
  int rc0 = sync(h);
  if (rc0) return rc0;
  double* out = ke;
  std::vector<double> blk;
  for (int64_t e = first; e < first + count; ++e) {
    const bool beam = e < P.n_beams;
    const int k = beam ? 2 : 4;
    const int64_t sb = beam ? 4 * e : 4 * (int64_t)P.n_beams + 16 * (e - P.n_beams);
    blk.resize((size_t)k * k * 36);
    CK(h, cudaMemcpy(blk.data(), P.stage + 36 * sb, blk.size() * sizeof(double), cudaMemcpyDeviceToHost));
    const int m = 6 * k;
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j)
        for (int a = 0; a < 6; ++a)
          for (int b = 0; b < 6; ++b) out[(6 * i + a) * m + 6 * j + b] = blk[(i * k + j) * 36 + 6 * a + b];
    out += m * m;
  }
  return SSO_OK;
}

int sso_export_dinv(sso_handle h, double* dinv) {
  ENTER(h);
  if (!h || !dinv) return SSO_E_INVALID;
  if (!h->assembled) FAIL(h, SSO_E_STATE, "export of dinv before sso_assemble");
  for (auto& pp : h->parts) {
    Part& P = *pp;
    CK(h, cudaMemcpy(dinv + 6 * (int64_t)(P.lm.own_begin - h->user_node_begin), P.dinv,
                     (size_t)P.ndof_own * sizeof(double), cudaMemcpyDeviceToHost));
  }
  return SSO_OK;
}

int sso_profile_enable(sso_handle h, int32_t on) {
  ENTER(h);
  if (!h) return SSO_E_INVALID;
  h->tm.on = on != 0;
  return SSO_OK;
}

int sso_profile_read(sso_handle h, const char* name, double* total_ms, int64_t* launches) {
  ENTER(h);
  if (!h || !name) return SSO_E_INVALID;
  static const char* names[F_COUNT] = {"element", "assemble", "spmv", "update", "grad", "reduce"};
  for (int k = 0; k < F_COUNT; ++k)
    if (std::strcmp(names[k], name) == 0) {
      if (total_ms) *total_ms = h->tm.total_ms[k];
      if (launches) *launches = h->tm.launches[k];
      return SSO_OK;
    }
  FAIL(h, SSO_E_INVALID, "unknown kernel family");
}

int sso_profile_reset(sso_handle h) {
  ENTER(h);
  if (!h) return SSO_E_INVALID;
  for (int k = 0; k < F_COUNT; ++k) {
    h->tm.total_ms[k] = 0;
    h->tm.launches[k] = 0;
  }
  return SSO_OK;
}

int64_t sso_launch_count(sso_handle h) { return h ? h->launches : 0; }

void sso_destroy(sso_handle h) {
  if (!h) return;
  int cur = -1;
  const bool sw = cudaGetDevice(&cur) == cudaSuccess && cur != h->device && cudaSetDevice(h->device) == cudaSuccess;
  cudaStreamSynchronize(h->stream);
  free_all(h);
  delete h;
  if (sw) cudaSetDevice(cur);
}

// ---------------------------------------------------------------------------
// Host-only partition queries (no GPU needed): used by the multi-process CPU
// tests of the partition logic.
// ---------------------------------------------------------------------------
int sso_local_pattern(const sso_mesh* mesh, const int32_t* ranges, int32_t n_parts, int32_t part,
                      int64_t* nnz, int64_t* row_ptr, int32_t* col_idx) {
  if (!mesh || !nnz || n_parts < 1 || part < 0 || part >= n_parts) return SSO_E_INVALID;
  std::vector<int32_t> rg = make_ranges(mesh->n_nodes, n_parts, ranges);
  LocalMesh L;
  std::string e = build_local_mesh(mesh->n_nodes, mesh->n_beams, mesh->beam_conn, mesh->n_quads,
                                   mesh->quad_conn, rg.data(), n_parts, part, L);
  if (!e.empty()) { g_create_err = e; return SSO_E_INVALID; }
  HostPattern T;
  e = build_pattern((int32_t)L.node_gid.size(), (int32_t)L.beam_gid.size(), L.beam_conn.data(),
                    (int32_t)L.quad_gid.size(), L.quad_conn.data(), T);
  if (!e.empty()) { g_create_err = e; return SSO_E_INVALID; }
  *nnz = 36 * T.node_ptr[L.n_own];
  if (!row_ptr && !col_idx) return SSO_OK;
  std::vector<int32_t> cols;
  int64_t row = 0;
  for (int32_t n = 0; n < L.n_own; ++n) {
    const int64_t b0 = T.node_ptr[n], deg = T.node_ptr[n + 1] - b0;
    cols.clear();
    for (int64_t k = 0; k < deg; ++k) cols.push_back(L.node_gid[T.node_col[b0 + k]]);
    std::sort(cols.begin(), cols.end());
    for (int a = 0; a < 6; ++a) {
      const int64_t start = 36 * b0 + 6 * a * deg;
      if (row_ptr) row_ptr[row + a] = start;
      if (col_idx)
        for (int64_t k = 0; k < deg; ++k)
          for (int b = 0; b < 6; ++b) col_idx[start + 6 * k + b] = 6 * cols[k] + b;
    }
    row += 6;
  }
  if (row_ptr) row_ptr[row] = *nnz;
  return SSO_OK;
}

int sso_halo_plan(const sso_mesh* mesh, const int32_t* ranges, int32_t n_parts, int32_t part,
                  int32_t* n_halo, int32_t* halo_gid, int32_t* n_nbrs, int32_t* nbr_part,
                  int32_t* send_count, int32_t* send_gid) {
  if (!mesh || !n_halo || !n_nbrs || n_parts < 1 || part < 0 || part >= n_parts) return SSO_E_INVALID;
  std::vector<int32_t> rg = make_ranges(mesh->n_nodes, n_parts, ranges);
  LocalMesh L;
  std::string e = build_local_mesh(mesh->n_nodes, mesh->n_beams, mesh->beam_conn, mesh->n_quads,
                                   mesh->quad_conn, rg.data(), n_parts, part, L);
  if (!e.empty()) { g_create_err = e; return SSO_E_INVALID; }
  *n_halo = (int32_t)L.node_gid.size() - L.n_own;
  *n_nbrs = (int32_t)L.nbrs.size();
  if (halo_gid)
    for (int32_t i = 0; i < *n_halo; ++i) halo_gid[i] = L.node_gid[L.n_own + i];
  int64_t off = 0;
  for (size_t k = 0; k < L.nbrs.size(); ++k) {
    if (nbr_part) nbr_part[k] = L.nbrs[k].part;
    if (send_count) send_count[k] = (int32_t)L.nbrs[k].send_local.size();
    if (send_gid)
      for (int32_t v : L.nbrs[k].send_local) send_gid[off++] = L.own_begin + v;
  }
  return SSO_OK;
}

}  // extern "C"
