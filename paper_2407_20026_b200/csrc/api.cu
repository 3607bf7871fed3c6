// C-ABI entry points (include/sso.h).  Host orchestration only: validation,
// pattern build (A0, pattern.cpp), device buffers, launch sequencing, the PCG
// chunk graphs and the exports.  Every step of the hot path runs in the
// kernels of elements.cu, assemble.cu, pcg.cu and grad.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "sso_internal.h"

using namespace sso;

struct sso_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t cap_stream = nullptr;
  sso_mem mem = SSO_MEM_HOST;
  double rtol = 1e-10;
  int64_t max_iter = 200000;
  double drill_alpha = 1e-3;
  int warm_start = 0;
  int check_every = 64;

  int32_t n_nodes = 0, n_beams = 0, n_quads = 0;
  int64_t ndof = 0, nnz = 0, n_blocks = 0, n_staged = 0, n_slots = 0;
  HostPattern pat;

  // device inputs
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
  // solver vectors
  double *f = nullptr, *fbc = nullptr, *xs = nullptr, *r = nullptr, *p = nullptr, *q = nullptr,
         *tmp = nullptr, *gu = nullptr, *gf = nullptr;
  double* partial = nullptr;
  CgState* st = nullptr;
  DevFlags* flags = nullptr;
  unsigned int* tickets = nullptr;
  double* scal = nullptr;  // device scalars [8]
  double *slot_partial = nullptr, *dxyz = nullptr, *dt = nullptr;
  // pinned host mirrors
  CgState* h_st = nullptr;
  double* h_scal = nullptr;
  CgState* h_chunk = nullptr;  // [2] pinned per-chunk state snapshots (polled)
  DevFlags* h_flags = nullptr;

  bool assembled = false, solved = false;
  cudaGraphExec_t chunk_exec = nullptr;   // K CG iterations
  cudaGraphExec_t prof_exec[2] = {nullptr, nullptr};  // same, with SpMV event nodes (slot 0/1)
  long long kernels_per_chunk = 0;
  std::vector<cudaEvent_t> chunk_ev[2];   // profiling: 2 per iteration per slot
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_done[2] = {nullptr, nullptr};

  Timers tm;
  long long launches = 0;
  std::string err;
};

static std::string g_create_err;

#define FAIL(h, code, msg)       \
  do {                           \
    (h)->err = (msg);            \
    return (code);               \
  } while (0)

#define CK(h, call)                                                                  \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      (h)->err = std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call; \
      return e_ == cudaErrorMemoryAllocation ? SSO_E_OOM : SSO_E_CUDA;               \
    }                                                                                \
  } while (0)

#define CKL(h)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess) {                                                            \
      (h)->err = std::string("CUDA launch error: ") + cudaGetErrorString(e_) + " (" +    \
                 last_launch_error() + ")";                                             \
      return SSO_E_CUDA;                                                                \
    }                                                                                   \
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

// copy a caller buffer (kind per h->mem) into a device buffer on h->stream
int copy_in(sso_ctx* h, double* dst, const double* src, int64_t n) {
  if (n <= 0) return SSO_OK;
  CK(h, cudaMemcpyAsync(dst, src, (size_t)n * sizeof(double),
                        h->mem == SSO_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                        h->stream));
  return SSO_OK;
}

int copy_out(sso_ctx* h, double* dst, const double* src, int64_t n) {
  if (n <= 0 || !dst) return SSO_OK;
  CK(h, cudaMemcpyAsync(dst, src, (size_t)n * sizeof(double),
                        h->mem == SSO_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                        h->stream));
  return SSO_OK;
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

int check_flags(sso_ctx* h) {
  CK(h, cudaMemcpyAsync(h->h_flags, h->flags, sizeof(DevFlags), cudaMemcpyDeviceToHost, h->stream));
  int rc = sync(h);
  if (rc) return rc;
  if (h->h_flags->degenerate_elem != INT_MAX) {
    int e = h->h_flags->degenerate_elem;
    char buf[256];
    if (e < 0) e = -e - 1;
    snprintf(buf, sizeof buf, "degenerate element %d (%s): zero length / zero normal / det J <= 0",
             e, e < h->n_beams ? "beam" : "quad");
    h->err = buf;
    return SSO_E_DEGENERATE;
  }
  if (h->h_flags->singular_dof != INT_MAX) {
    int d = h->h_flags->singular_dof;
    char buf[256];
    snprintf(buf, sizeof buf, "singular: free DOF %d (node %d, component %d) has diagonal <= 0", d,
             d / 6, d % 6);
    h->err = buf;
    return SSO_E_SINGULAR;
  }
  return SSO_OK;
}

int reset_flags(sso_ctx* h) {
  h->h_flags->degenerate_elem = INT_MAX;
  h->h_flags->singular_dof = INT_MAX;
  CK(h, cudaMemcpyAsync(h->flags, h->h_flags, sizeof(DevFlags), cudaMemcpyHostToDevice, h->stream));
  return SSO_OK;
}

// Capture K = check_every CG iterations into a graph.  prof_slot >= 0 adds
// external event-record nodes around every PROF_EVERY-th SpMV (events of that
// slot): a live sample of the SpMV launch duration that costs < 0.5 % of the step.
constexpr int PROF_EVERY = 16;
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
  long long g0 = g_launches;
  CK(h, cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < K; ++i) {
    const bool rec = prof_slot >= 0 && (i % PROF_EVERY) == 0;
    if (rec)
      cudaEventRecordWithFlags(h->chunk_ev[prof_slot][2 * i], h->cap_stream, cudaEventRecordExternal);
    launch_spmv_dot(h->cap_stream, h->n_nodes, h->node_ptr, h->node_col, h->vals, h->p, h->q,
                    h->partial, h->st);
    if (rec)
      cudaEventRecordWithFlags(h->chunk_ev[prof_slot][2 * i + 1], h->cap_stream, cudaEventRecordExternal);
    launch_cg_update(h->cap_stream, (int)h->ndof, h->dinv, h->xs, h->r, h->p, h->q, h->partial, h->st);
    launch_cg_pupdate(h->cap_stream, (int)h->ndof, h->dinv, h->r, h->p, h->st);
  }
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
  h->kernels_per_chunk = g_launches - g0;
  g_launches = g0;  // captured launches are counted per replay
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

int free_all(sso_ctx* h) {
  void* ptrs[] = {h->x, h->y, h->z, h->beam_conn, h->quad_conn, h->A, h->Iy, h->Iz, h->J, h->t,
                  h->E, h->nu, h->G, h->fixed_mask, h->node_ptr, h->node_col, h->contrib_ptr,
                  h->contrib, h->inc_ptr, h->inc_slot, h->stage, h->vals, h->dinv, h->f, h->fbc,
                  h->xs, h->r, h->p, h->q, h->tmp, h->gu, h->gf, h->partial, h->st, h->flags,
                  h->tickets, h->scal, h->slot_partial, h->dxyz, h->dt};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->h_st) cudaFreeHost(h->h_st);
  if (h->h_scal) cudaFreeHost(h->h_scal);
  if (h->h_chunk) cudaFreeHost(h->h_chunk);
  if (h->h_flags) cudaFreeHost(h->h_flags);
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
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  return SSO_OK;
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

}  // namespace

extern "C" {

int sso_options_default(sso_options* o) {
  if (!o) return SSO_E_INVALID;
  o->rtol = 1e-10;
  o->max_iter = 200000;
  o->drill_alpha = 1e-3;
  o->warm_start = 0;
  o->check_every = 64;
  o->mem = SSO_MEM_HOST;
  o->cuda_stream = nullptr;
  o->device = -1;
  return SSO_OK;
}

const char* sso_last_error(sso_handle h) { return h ? h->err.c_str() : g_create_err.c_str(); }

int sso_create(const sso_mesh* mesh, const sso_sections* sec, const sso_materials* mat,
               const sso_supports* sup, const sso_options* opt, sso_handle* out) {
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
  sso_ctx* h = new sso_ctx();
  auto bail = [&](int code) {
    g_create_err = h->err;
    free_all(h);
    delete h;
    return code;
  };
  if (o.device >= 0) {
    if (cudaSetDevice(o.device) != cudaSuccess) { h->err = "cudaSetDevice failed"; return bail(SSO_E_CUDA); }
  }
  if (cudaGetDevice(&h->device) != cudaSuccess) { h->err = "no CUDA device"; return bail(SSO_E_CUDA); }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { h->err = "no CUDA device"; return bail(SSO_E_CUDA); }
  h->rtol = o.rtol;
  h->max_iter = o.max_iter;
  h->drill_alpha = o.drill_alpha;
  h->warm_start = o.warm_start;
  h->check_every = o.check_every;
  h->mem = o.mem;
  if (o.cuda_stream) {
    h->stream = (cudaStream_t)o.cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) { h->err = "stream create failed"; return bail(SSO_E_CUDA); }
    h->own_stream = true;
  }
  if (cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking) != cudaSuccess) { h->err = "stream create failed"; return bail(SSO_E_CUDA); }

  h->n_nodes = mesh->n_nodes;
  h->n_beams = mesh->n_beams;
  h->n_quads = mesh->n_quads;
  h->ndof = 6 * (int64_t)mesh->n_nodes;
  std::string perr = build_pattern(mesh->n_nodes, mesh->n_beams, mesh->beam_conn, mesh->n_quads,
                                   mesh->quad_conn, h->pat);
  if (!perr.empty()) { h->err = perr; return bail(SSO_E_INVALID); }
  h->n_blocks = h->pat.n_blocks();
  h->nnz = h->pat.nnz();
  h->n_staged = h->pat.n_staged_blocks();
  h->n_slots = 2 * (int64_t)h->n_beams + 4 * (int64_t)h->n_quads;
  const int64_t ne = (int64_t)h->n_beams + h->n_quads;

  // host-side derived inputs: G (beams), OR-merged support masks
  std::vector<double> G((size_t)ne);
  for (int64_t e = 0; e < ne; ++e) G[e] = mat->G ? mat->G[e] : mat->E[e] / (2.0 * (1.0 + mat->nu[e]));
  std::vector<uint8_t> mask((size_t)h->n_nodes, 0);
  for (int32_t k = 0; k < sup->n; ++k) mask[sup->node[k]] |= (uint8_t)(sup->mask6[k] & 63);

  int r;
#define UP(dst, src, n) if ((r = upload(h, &h->dst, src, n))) return bail(r)
#define AL(dst, n) if ((r = dalloc(h, &h->dst, n))) return bail(r)
  UP(x, mesh->x, h->n_nodes);
  UP(y, mesh->y, h->n_nodes);
  UP(z, mesh->z, h->n_nodes);
  UP(beam_conn, mesh->beam_conn, 2 * (int64_t)h->n_beams);
  UP(quad_conn, mesh->quad_conn, 4 * (int64_t)h->n_quads);
  UP(A, sec->A, h->n_beams);
  UP(Iy, sec->Iy, h->n_beams);
  UP(Iz, sec->Iz, h->n_beams);
  UP(J, sec->J, h->n_beams);
  UP(t, sec->t, h->n_quads);
  UP(E, mat->E, ne);
  UP(nu, mat->nu, ne);
  UP(G, G.data(), ne);
  UP(fixed_mask, mask.data(), h->n_nodes);
  UP(node_ptr, h->pat.node_ptr.data(), h->n_nodes + 1);
  UP(node_col, h->pat.node_col.data(), h->n_blocks);
  UP(contrib_ptr, h->pat.contrib_ptr.data(), h->n_blocks + 1);
  UP(contrib, h->pat.contrib.data(), h->n_staged);
  UP(inc_ptr, h->pat.inc_ptr.data(), h->n_nodes + 1);
  UP(inc_slot, h->pat.inc_slot.data(), h->n_slots);
  AL(stage, 36 * h->n_staged);
  AL(vals, h->nnz);
  AL(dinv, h->ndof);
  AL(f, h->ndof);
  AL(fbc, h->ndof);
  AL(xs, h->ndof);
  AL(r, h->ndof);
  AL(p, h->ndof);
  AL(q, h->ndof);
  AL(tmp, h->ndof);
  AL(gu, h->ndof);
  AL(gf, h->ndof);
  AL(partial, 4 * (int64_t)cg_grid() * 4);
  AL(st, 1);
  AL(flags, 1);
  AL(tickets, 16);
  AL(scal, 8);
  AL(slot_partial, 3 * std::max<int64_t>(h->n_slots, 1));
  AL(dxyz, 3 * (int64_t)h->n_nodes);
  AL(dt, std::max<int32_t>(h->n_quads, 1));
#undef UP
#undef AL
  if (cudaMemset(h->tickets, 0, 16 * sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(h->st, 0, sizeof(CgState)) != cudaSuccess ||
      cudaMemset(h->xs, 0, h->ndof * sizeof(double)) != cudaSuccess) { h->err = "memset failed"; return bail(SSO_E_CUDA); }
  if (cudaMallocHost(&h->h_st, sizeof(CgState)) != cudaSuccess ||
      cudaMallocHost(&h->h_scal, 8 * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&h->h_chunk, 2 * sizeof(CgState)) != cudaSuccess ||
      cudaMallocHost(&h->h_flags, sizeof(DevFlags)) != cudaSuccess) { h->err = "cudaMallocHost failed"; return bail(SSO_E_OOM); }
  cudaEventCreate(&h->ev_a);
  cudaEventCreate(&h->ev_b);
  cudaEventCreateWithFlags(&h->ev_done[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->ev_done[1], cudaEventDisableTiming);
  // the pattern's large contributor / incidence arrays are only needed on the device
  h->pat.contrib.clear();
  h->pat.contrib.shrink_to_fit();
  h->pat.inc_slot.clear();
  h->pat.inc_slot.shrink_to_fit();
  *out = h;
  return SSO_OK;
}

int sso_set_stream(sso_handle h, void* cuda_stream, sso_mem mem) {
  if (!h) return SSO_E_INVALID;
  if (cuda_stream) {
    if (h->own_stream) cudaStreamDestroy(h->stream);
    h->own_stream = false;
    h->stream = (cudaStream_t)cuda_stream;
  }
  h->mem = mem;
  return SSO_OK;
}

int sso_set_design(sso_handle h, const double* x, const double* y, const double* z, const double* t) {
  if (!h) return SSO_E_INVALID;
  int rc;
  if (x && (rc = copy_in(h, h->x, x, h->n_nodes))) return rc;
  if (y && (rc = copy_in(h, h->y, y, h->n_nodes))) return rc;
  if (z && (rc = copy_in(h, h->z, z, h->n_nodes))) return rc;
  if (t && (rc = copy_in(h, h->t, t, h->n_quads))) return rc;
  h->assembled = false;
  h->solved = false;
  return sync(h);
}

int sso_assemble(sso_handle h) {
  if (!h) return SSO_E_INVALID;
  int rc = reset_flags(h);
  if (rc) return rc;
  {
    Scope sc(h, F_ELEMENT);
    launch_beam_elements(h->stream, h->n_beams, h->x, h->y, h->z, h->beam_conn, h->A, h->Iy, h->Iz,
                         h->J, h->E, h->G, h->stage, h->flags);
    launch_quad_elements(h->stream, h->n_quads, h->x, h->y, h->z, h->quad_conn, h->t,
                         h->E + h->n_beams, h->nu + h->n_beams, h->drill_alpha,
                         h->stage + 36 * 4 * (int64_t)h->n_beams, h->flags);
  }
  {
    Scope sc(h, F_ASSEMBLE);
    launch_assemble(h->stream, h->n_nodes, h->node_ptr, h->node_col, h->contrib_ptr, h->contrib,
                    h->stage, h->fixed_mask, h->vals, h->dinv, h->flags);
  }
  CKL(h);
  rc = check_flags(h);
  if (rc) return rc;
  h->assembled = true;
  h->solved = false;
  return SSO_OK;
}

int sso_solve(sso_handle h, const double* f, double* u, sso_solve_info* info) {
  if (!h || !f || !u) {
    if (h) h->err = "null argument";
    return SSO_E_INVALID;
  }
  if (!h->assembled) FAIL(h, SSO_E_STATE, "sso_solve before sso_assemble");
  int rc;
  if ((rc = copy_in(h, h->f, f, h->ndof))) return rc;
  const int warm = h->warm_start ? 1 : 0;
  if (warm) {
    if ((rc = copy_in(h, h->xs, u, h->ndof))) return rc;
    {
      Scope sc(h, F_UPDATE);
      launch_zero_fixed(h->stream, (int)h->ndof, h->fixed_mask, h->xs);
    }
    Scope sc(h, F_SPMV);
    launch_spmv(h->stream, h->n_nodes, h->node_ptr, h->node_col, h->vals, h->xs, h->tmp);
  }
  std::memset(h->h_st, 0, sizeof(CgState));
  h->h_st->tol2 = h->rtol * h->rtol;
  h->h_st->max_iter = h->max_iter;
  CK(h, cudaMemcpyAsync(h->st, h->h_st, sizeof(CgState), cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaEventRecord(h->ev_a, h->stream));
  {
    Scope sc(h, F_UPDATE);
    launch_cg_init(h->stream, (int)h->ndof, h->f, h->fixed_mask, h->dinv, h->fbc, h->xs, h->r, h->p,
                   h->partial, h->st, warm, h->tmp);
  }
  const bool prof = h->tm.on;
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
  // profiling on, slot-alternating graphs carry event nodes around every SpMV and
  // the elapsed times of the iterations that actually ran are accumulated.
  const int64_t max_chunks = (h->max_iter + h->check_every - 1) / h->check_every + 1;
  int64_t launched = 0;
  auto launch_chunk = [&](int slot) -> int {
    CK(h, cudaGraphLaunch(prof ? h->prof_exec[slot] : h->chunk_exec, h->stream));
    h->launches += h->kernels_per_chunk;
    CK(h, cudaMemcpyAsync(&h->h_chunk[slot], h->st, sizeof(CgState), cudaMemcpyDeviceToHost,
                          h->stream));
    CK(h, cudaEventRecord(h->ev_done[slot], h->stream));
    ++launched;
    return SSO_OK;
  };
  long long iters_before = 0;
  if ((rc = launch_chunk(0))) return rc;
  for (int64_t k = 0;; ++k) {
    const int slot = (int)(k & 1);
    if (launched < max_chunks && (rc = launch_chunk(1 - slot))) return rc;
    CK(h, cudaEventSynchronize(h->ev_done[slot]));
    const CgState& S = h->h_chunk[slot];
    if (prof) {
      long long ran = S.iter - iters_before;
      if (S.done && S.status == SSO_E_NOT_SPD && ran < h->check_every) ran += 1;
      iters_before = S.iter;
      for (long long i = 0; i < std::min<long long>(ran, h->check_every); i += PROF_EVERY) {
        float ms = 0.f;
        CK(h, cudaEventElapsedTime(&ms, h->chunk_ev[slot][2 * i], h->chunk_ev[slot][2 * i + 1]));
        h->tm.total_ms[F_SPMV] += ms;
        h->tm.launches[F_SPMV] += 1;
      }
    }
    if (S.done || launched == k + 1) break;
  }
  CK(h, cudaEventRecord(h->ev_b, h->stream));
  // true residual |f_bc - K x| / |f_bc|
  {
    long long g1 = g_launches;
    launch_spmv(h->stream, h->n_nodes, h->node_ptr, h->node_col, h->vals, h->xs, h->tmp);
    launch_residual_norm(h->stream, (int)h->ndof, h->fbc, h->tmp, h->partial, h->tickets + 2, h->scal);
    h->launches += g_launches - g1;
  }
  CK(h, cudaMemcpyAsync(h->h_scal, h->scal, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaMemcpyAsync(h->h_st, h->st, sizeof(CgState), cudaMemcpyDeviceToHost, h->stream));
  if ((rc = copy_out(h, u, h->xs, h->ndof))) return rc;
  if ((rc = sync(h))) return rc;
  CKL(h);
  const CgState& S = *h->h_st;
  int status = S.done ? S.status : SSO_E_NOT_CONVERGED;
  if (info) {
    info->iters = S.iter;
    info->rel_res = S.ff > 0 ? std::sqrt(S.rr / S.ff) : 0.0;
    info->true_rel_res = S.ff > 0 ? std::sqrt(h->h_scal[0] / S.ff) : 0.0;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, h->ev_a, h->ev_b) != cudaSuccess) (void)cudaGetLastError();
    info->ms = ms;
    info->status = status;
  }
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

static int grad_impl(sso_ctx* h, sso_objective obj, const double* dF, const double* dU, double* C,
                     double* dC_dxyz, double* dC_dt) {
  const double s = (obj == SSO_OBJ_STRAIN_ENERGY) ? 0.5 : 1.0;
  {
    Scope sc(h, F_REDUCE);
    launch_dot(h->stream, (int)h->ndof, dF, dU, s, h->partial, h->tickets + 3, h->scal + 1);
  }
  {
    Scope sc(h, F_GRAD);
    launch_beam_grad(h->stream, h->n_beams, h->x, h->y, h->z, h->beam_conn, h->A, h->Iy, h->Iz, h->J,
                     h->E, h->G, dU, s, h->slot_partial);
    launch_quad_grad(h->stream, h->n_beams, h->n_quads, h->x, h->y, h->z, h->quad_conn, h->t, h->E,
                     h->nu, h->drill_alpha, dU, s, h->slot_partial, h->dt);
  }
  {
    Scope sc(h, F_REDUCE);
    launch_node_reduce(h->stream, h->n_nodes, h->inc_ptr, h->inc_slot, h->slot_partial, h->dxyz);
  }
  CKL(h);
  int rc;
  if (C) {
    CK(h, cudaMemcpyAsync(h->h_scal + 1, h->scal + 1, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  }
  if (dC_dxyz && (rc = copy_out(h, dC_dxyz, h->dxyz, 3 * (int64_t)h->n_nodes))) return rc;
  if (dC_dt && (rc = copy_out(h, dC_dt, h->dt, h->n_quads))) return rc;
  if ((rc = sync(h))) return rc;
  if (C) {
    if (h->mem == SSO_MEM_HOST) {
      *C = h->h_scal[1];
    } else {
      CK(h, cudaMemcpy(C, h->scal + 1, sizeof(double), cudaMemcpyDeviceToDevice));
    }
  }
  return SSO_OK;
}

int sso_grad(sso_handle h, sso_objective obj, double* C, double* dC_dxyz, double* dC_dt) {
  if (!h) return SSO_E_INVALID;
  if (obj != SSO_OBJ_COMPLIANCE && obj != SSO_OBJ_STRAIN_ENERGY) FAIL(h, SSO_E_INVALID, "unknown objective");
  if (!h->solved) FAIL(h, SSO_E_STATE, "sso_grad before a successful sso_solve");
  return grad_impl(h, obj, h->f, h->xs, C, dC_dxyz, dC_dt);
}

int sso_grad_at(sso_handle h, sso_objective obj, const double* f, const double* u, double* C,
                double* dC_dxyz, double* dC_dt) {
  if (!h || !f || !u) return SSO_E_INVALID;
  if (obj != SSO_OBJ_COMPLIANCE && obj != SSO_OBJ_STRAIN_ENERGY) FAIL(h, SSO_E_INVALID, "unknown objective");
  int rc;
  if ((rc = copy_in(h, h->gf, f, h->ndof))) return rc;
  if ((rc = copy_in(h, h->gu, u, h->ndof))) return rc;
  return grad_impl(h, obj, h->gf, h->gu, C, dC_dxyz, dC_dt);
}

int sso_spmv(sso_handle h, const double* xin, double* yout) {
  if (!h || !xin || !yout) return SSO_E_INVALID;
  if (!h->assembled) FAIL(h, SSO_E_STATE, "sso_spmv before sso_assemble");
  int rc;
  if ((rc = copy_in(h, h->gu, xin, h->ndof))) return rc;
  {
    Scope sc(h, F_SPMV);
    launch_spmv(h->stream, h->n_nodes, h->node_ptr, h->node_col, h->vals, h->gu, h->tmp);
  }
  CKL(h);
  if ((rc = copy_out(h, yout, h->tmp, h->ndof))) return rc;
  return sync(h);
}

int sso_sizes(sso_handle h, int64_t* ndof, int64_t* nnz, int64_t* n_blocks) {
  if (!h) return SSO_E_INVALID;
  if (ndof) *ndof = h->ndof;
  if (nnz) *nnz = h->nnz;
  if (n_blocks) *n_blocks = h->n_blocks;
  return SSO_OK;
}

int sso_export_csr(sso_handle h, int64_t* row_ptr, int32_t* col_idx, double* vals) {
  if (!h) return SSO_E_INVALID;
  const HostPattern& P = h->pat;
  if (row_ptr || col_idx) {
    for (int32_t n = 0; n < h->n_nodes; ++n) {
      const int64_t b0 = P.node_ptr[n];
      const int64_t deg = P.node_ptr[n + 1] - b0;
      for (int a = 0; a < 6; ++a) {
        const int64_t start = 36 * b0 + 6 * a * deg;
        if (row_ptr) row_ptr[6 * (int64_t)n + a] = start;
        if (col_idx)
          for (int64_t k = 0; k < deg; ++k)
            for (int b = 0; b < 6; ++b) col_idx[start + 6 * k + b] = 6 * P.node_col[b0 + k] + b;
      }
    }
    if (row_ptr) row_ptr[h->ndof] = h->nnz;
  }
  if (vals) {
    if (!h->assembled) FAIL(h, SSO_E_STATE, "export of values before sso_assemble");
    CK(h, cudaMemcpy(vals, h->vals, h->nnz * sizeof(double), cudaMemcpyDeviceToHost));
  }
  return SSO_OK;
}

int sso_export_scatter(sso_handle h, int32_t* block_rank) {
  if (!h || !block_rank) return SSO_E_INVALID;
  std::memcpy(block_rank, h->pat.block_rank.data(), h->pat.block_rank.size() * sizeof(int32_t));
  return SSO_OK;
}

int sso_export_ke(sso_handle h, int64_t first, int64_t count, double* ke) {
  if (!h || !ke) return SSO_E_INVALID;
  const int64_t ne = (int64_t)h->n_beams + h->n_quads;
  if (first < 0 || count < 0 || first + count > ne) FAIL(h, SSO_E_INVALID, "element range out of bounds");
  if (!h->assembled) FAIL(h, SSO_E_STATE, "export of K_e before sso_assemble");
  double* out = ke;
  std::vector<double> blk;
  for (int64_t e = first; e < first + count; ++e) {
    const bool beam = e < h->n_beams;
    const int k = beam ? 2 : 4;
    const int64_t sb = beam ? 4 * e : 4 * (int64_t)h->n_beams + 16 * (e - h->n_beams);
    blk.resize((size_t)k * k * 36);
    CK(h, cudaMemcpy(blk.data(), h->stage + 36 * sb, blk.size() * sizeof(double), cudaMemcpyDeviceToHost));
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
  if (!h || !dinv) return SSO_E_INVALID;
  if (!h->assembled) FAIL(h, SSO_E_STATE, "export of dinv before sso_assemble");
  CK(h, cudaMemcpy(dinv, h->dinv, h->ndof * sizeof(double), cudaMemcpyDeviceToHost));
  return SSO_OK;
}

int sso_profile_enable(sso_handle h, int32_t on) {
  if (!h) return SSO_E_INVALID;
  h->tm.on = on != 0;
  return SSO_OK;
}

int sso_profile_read(sso_handle h, const char* name, double* total_ms, int64_t* launches) {
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
  cudaStreamSynchronize(h->stream);
  free_all(h);
  delete h;
}

}  // extern "C"
