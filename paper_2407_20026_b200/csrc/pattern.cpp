// A0 — CSR pattern builder (host C++), SURVEY.md §8(a) A0.
//
// `element_K_*_indices` return the global rows/columns of each
// element entry; PAPER.md:83 — the global K is a sparse matrix whose duplicate
// element entries are summed.  This builder fixes that sparse structure once
// per connectivity (reading c8: structural pattern incl. zeros; columns
// ascending; contributors in ascending (e, i, j)):
//   * node graph: m in adj(n) iff n and m share an element (incl. n itself);
//   * block rank map: rank[e][i][j] = position of node j in adj(node i);
//   * per node-block contributor lists of staged element blocks, ascending e;
//   * node -> element-node incidence (for the gradient node reduction).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "sso_internal.h"

namespace sso {

std::string build_pattern(int32_t n_nodes, int32_t n_beams, const int32_t* beam_conn,
                          int32_t n_quads, const int32_t* quad_conn, HostPattern& P) {
  P.n_nodes = n_nodes;
  P.n_beams = n_beams;
  P.n_quads = n_quads;
  const int64_t n_slots = 2 * (int64_t)n_beams + 4 * (int64_t)n_quads;

  // node -> element-node incidence, slots ascending in e (beams first, then quads)
  P.inc_ptr.assign((size_t)n_nodes + 1, 0);
  for (int32_t e = 0; e < n_beams; ++e)
    for (int i = 0; i < 2; ++i) P.inc_ptr[(size_t)beam_conn[2 * e + i] + 1]++;
  for (int32_t q = 0; q < n_quads; ++q)
    for (int i = 0; i < 4; ++i) P.inc_ptr[(size_t)quad_conn[4 * (int64_t)q + i] + 1]++;
  for (int32_t n = 0; n < n_nodes; ++n) P.inc_ptr[n + 1] += P.inc_ptr[n];
  P.inc_slot.assign((size_t)n_slots, 0);
  {
    std::vector<int64_t> fill(P.inc_ptr.begin(), P.inc_ptr.end() - 1);
    for (int32_t e = 0; e < n_beams; ++e)
      for (int i = 0; i < 2; ++i) P.inc_slot[fill[beam_conn[2 * e + i]]++] = 2 * e + i;
    for (int32_t q = 0; q < n_quads; ++q)
      for (int i = 0; i < 4; ++i)
        P.inc_slot[fill[quad_conn[4 * (int64_t)q + i]]++] = 2 * n_beams + 4 * q + i;
  }
  auto slot_node = [&](int32_t slot) -> int32_t {
    if (slot < 2 * n_beams) return beam_conn[slot];
    int64_t s = slot - 2 * (int64_t)n_beams;
    return quad_conn[s];
  };
  auto slot_elem_nodes = [&](int32_t slot, int32_t* out) -> int {
    if (slot < 2 * n_beams) {
      int32_t e = slot / 2;
      out[0] = beam_conn[2 * e];
      out[1] = beam_conn[2 * e + 1];
      return 2;
    }
    int64_t q = (slot - 2 * (int64_t)n_beams) / 4;
    for (int i = 0; i < 4; ++i) out[i] = quad_conn[4 * q + i];
    return 4;
  };
  (void)slot_node;

  // node graph: sorted unique neighbours of every node (incl. itself)
  P.node_ptr.assign((size_t)n_nodes + 1, 0);
  std::vector<std::vector<int32_t>> adj((size_t)n_nodes);
  {
    std::vector<int32_t> buf;
    int32_t en[4];
    for (int32_t n = 0; n < n_nodes; ++n) {
      buf.clear();
      buf.push_back(n);
      for (int64_t k = P.inc_ptr[n]; k < P.inc_ptr[n + 1]; ++k) {
        int c = slot_elem_nodes(P.inc_slot[k], en);
        for (int i = 0; i < c; ++i) buf.push_back(en[i]);
      }
      std::sort(buf.begin(), buf.end());
      buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
      adj[n] = buf;
      P.node_ptr[n + 1] = P.node_ptr[n] + (int64_t)buf.size();
    }
  }
  const int64_t nb = P.node_ptr[n_nodes];
  if (36 * nb > ((int64_t)1 << 62)) return "pattern too large";
  P.node_col.resize((size_t)nb);
  for (int32_t n = 0; n < n_nodes; ++n)
    std::memcpy(&P.node_col[P.node_ptr[n]], adj[n].data(), adj[n].size() * sizeof(int32_t));
  adj.clear();
  adj.shrink_to_fit();

  auto rank_of = [&](int32_t n, int32_t m) -> int32_t {
    const int32_t* b = &P.node_col[P.node_ptr[n]];
    const int32_t* e = &P.node_col[P.node_ptr[n + 1]];
    const int32_t* it = std::lower_bound(b, e, m);
    return (int32_t)(it - b);
  };

  // block rank map (beams [Eb][4], quads [Eq][16]) and contributor counts
  P.block_rank.resize((size_t)(4 * (int64_t)n_beams + 16 * (int64_t)n_quads));
  P.contrib_ptr.assign((size_t)nb + 1, 0);
  for (int32_t e = 0; e < n_beams; ++e)
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) {
        int32_t ni = beam_conn[2 * e + i], nj = beam_conn[2 * e + j];
        int32_t r = rank_of(ni, nj);
        P.block_rank[4 * (int64_t)e + 2 * i + j] = r;
        P.contrib_ptr[P.node_ptr[ni] + r + 1]++;
      }
  for (int32_t q = 0; q < n_quads; ++q)
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        int32_t ni = quad_conn[4 * (int64_t)q + i], nj = quad_conn[4 * (int64_t)q + j];
        int32_t r = rank_of(ni, nj);
        P.block_rank[4 * (int64_t)n_beams + 16 * (int64_t)q + 4 * i + j] = r;
        P.contrib_ptr[P.node_ptr[ni] + r + 1]++;
      }
  for (int64_t b = 0; b < nb; ++b) P.contrib_ptr[b + 1] += P.contrib_ptr[b];
  const int64_t nstaged = P.n_staged_blocks();
  if (nstaged >= ((int64_t)1 << 31)) return "too many element blocks for int32 contributor ids";
  P.contrib.resize((size_t)nstaged);
  {
    // filling in ascending (e, i, j) keeps every contributor list ascending
    std::vector<int64_t> fill(P.contrib_ptr.begin(), P.contrib_ptr.end() - 1);
    for (int32_t e = 0; e < n_beams; ++e)
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
          int32_t ni = beam_conn[2 * e + i];
          int64_t blk = P.node_ptr[ni] + P.block_rank[4 * (int64_t)e + 2 * i + j];
          P.contrib[fill[blk]++] = 4 * e + 2 * i + j;
        }
    for (int32_t q = 0; q < n_quads; ++q)
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
          int32_t ni = quad_conn[4 * (int64_t)q + i];
          int64_t blk = P.node_ptr[ni] + P.block_rank[4 * (int64_t)n_beams + 16 * (int64_t)q + 4 * i + j];
          P.contrib[fill[blk]++] = (int32_t)(4 * (int64_t)n_beams + 16 * (int64_t)q + 4 * i + j);
        }
  }
  return std::string();
}

void build_upper(const HostPattern& P, const int32_t* beam_conn, const int32_t* quad_conn,
                 UpperPattern& U) {
  const int32_t nn = P.n_nodes;
  U = UpperPattern();
  U.uptr.assign((size_t)nn + 1, 0);
  std::vector<int32_t> first_upper((size_t)nn);  // position of n itself in adj(n)
  for (int32_t n = 0; n < nn; ++n) {
    const int64_t b0 = P.node_ptr[n], b1 = P.node_ptr[n + 1];
    int64_t k = b0;
    while (k < b1 && P.node_col[k] < n) ++k;
    first_upper[n] = (int32_t)(k - b0);
    U.uptr[n + 1] = U.uptr[n] + (b1 - k);
  }
  U.ucol.resize((size_t)U.uptr[nn]);
  for (int32_t n = 0; n < nn; ++n) {
    const int64_t src = P.node_ptr[n] + first_upper[n];
    std::copy(P.node_col.begin() + src, P.node_col.begin() + P.node_ptr[n + 1], U.ucol.begin() + U.uptr[n]);
  }
  // element block ranks in the upper lists, and the upper contributor lists
  U.urank.resize(P.block_rank.size());
  U.ucontrib_ptr.assign((size_t)U.uptr[nn] + 1, 0);
  auto elem = [&](int64_t e, int& k, const int32_t*& c, int64_t& base) {
    if (e < P.n_beams) { k = 2; c = beam_conn + 2 * e; base = 4 * e; }
    else { const int64_t q = e - P.n_beams; k = 4; c = quad_conn + 4 * q; base = 4 * (int64_t)P.n_beams + 16 * q; }
  };
  const int64_t ne = (int64_t)P.n_beams + P.n_quads;
  for (int64_t e = 0; e < ne; ++e) {
    int k; const int32_t* c; int64_t base;
    elem(e, k, c, base);
    for (int i = 0; i < k; ++i)
      for (int jj = 0; jj < k; ++jj) {
        const int32_t ni = c[i], nj = c[jj];
        int32_t r = -1;
        if (nj >= ni) {
          r = P.block_rank[base + i * k + jj] - first_upper[ni];
          U.ucontrib_ptr[U.uptr[ni] + r + 1]++;
        }
        U.urank[base + i * k + jj] = r;
      }
  }
  for (int64_t b = 0; b < U.uptr[nn]; ++b) U.ucontrib_ptr[b + 1] += U.ucontrib_ptr[b];
  U.ucontrib.resize((size_t)U.ucontrib_ptr[U.uptr[nn]]);
  {
    std::vector<int64_t> fill(U.ucontrib_ptr.begin(), U.ucontrib_ptr.end() - 1);
    for (int64_t e = 0; e < ne; ++e) {
      int k; const int32_t* c; int64_t base;
      elem(e, k, c, base);
      for (int i = 0; i < k; ++i)
        for (int jj = 0; jj < k; ++jj) {
          const int32_t r = U.urank[base + i * k + jj];
          if (r >= 0) U.ucontrib[fill[U.uptr[c[i]] + r]++] = (int32_t)(base + i * k + jj);
        }
    }
  }
  // incoming blocks per node (lptr), ascending source node
  U.lptr.assign((size_t)nn + 1, 0);
  for (int32_t n = 0; n < nn; ++n)
    for (int64_t k = U.uptr[n] + 1; k < U.uptr[n + 1]; ++k) U.lptr[U.ucol[k] + 1]++;
  for (int32_t n = 0; n < nn; ++n) U.lptr[n + 1] += U.lptr[n];
  // pull lists (storage 3): the same incoming blocks as (source node, upper block index)
  U.lpull.resize(2 * (size_t)U.lptr[nn]);
  {
    std::vector<int64_t> fill(U.lptr.begin(), U.lptr.end() - 1);
    for (int32_t n = 0; n < nn; ++n)
      for (int64_t k = U.uptr[n] + 1; k < U.uptr[n + 1]; ++k) {
        const int64_t at = fill[U.ucol[k]]++;
        U.lpull[2 * at] = n;
        U.lpull[2 * at + 1] = (int32_t)k;
      }
  }
}

}  // namespace sso

namespace sso {

namespace {

int32_t owner_of(const int32_t* ranges, int32_t n_parts, int32_t node) {
  // ranges ascending; binary search for the part containing node
  int32_t lo = 0, hi = n_parts - 1;
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) / 2;
    if (ranges[mid] <= node) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Halo node set of part p (sorted by (owner, gid)) and its local element lists.
void part_elements(int32_t n_nodes, int32_t n_beams, const int32_t* beam_conn, int32_t n_quads,
                   const int32_t* quad_conn, int32_t b, int32_t e, std::vector<int32_t>& beams,
                   std::vector<int32_t>& quads) {
  (void)n_nodes;
  beams.clear();
  quads.clear();
  for (int32_t k = 0; k < n_beams; ++k) {
    const int32_t a = beam_conn[2 * k], c = beam_conn[2 * k + 1];
    if ((a >= b && a < e) || (c >= b && c < e)) beams.push_back(k);
  }
  for (int32_t k = 0; k < n_quads; ++k) {
    const int32_t* q = quad_conn + 4 * (int64_t)k;
    bool own = false;
    for (int i = 0; i < 4; ++i) own |= (q[i] >= b && q[i] < e);
    if (own) quads.push_back(k);
  }
}

std::vector<int32_t> halo_nodes(const int32_t* ranges, int32_t n_parts, int32_t p,
                                const int32_t* beam_conn, const int32_t* quad_conn,
                                const std::vector<int32_t>& beams, const std::vector<int32_t>& quads) {
  const int32_t b = ranges[p], e = ranges[p + 1];
  std::vector<int32_t> h;
  for (int32_t k : beams)
    for (int i = 0; i < 2; ++i) {
      const int32_t n = beam_conn[2 * k + i];
      if (n < b || n >= e) h.push_back(n);
    }
  for (int32_t k : quads)
    for (int i = 0; i < 4; ++i) {
      const int32_t n = quad_conn[4 * (int64_t)k + i];
      if (n < b || n >= e) h.push_back(n);
    }
  std::sort(h.begin(), h.end());
  h.erase(std::unique(h.begin(), h.end()), h.end());
  // order by (owner part, gid): gids are sorted and parts are contiguous ranges, so
  // sorting by gid already groups by owner in ascending part order
  (void)n_parts;
  return h;
}

}  // namespace

std::string build_local_mesh(int32_t n_nodes, int32_t n_beams, const int32_t* beam_conn,
                             int32_t n_quads, const int32_t* quad_conn, const int32_t* ranges,
                             int32_t n_parts, int32_t part, LocalMesh& L) {
  if (n_parts < 1 || part < 0 || part >= n_parts) return "bad part index";
  if (ranges[0] != 0 || ranges[n_parts] != n_nodes) return "part ranges must cover [0, n_nodes)";
  for (int32_t p = 0; p < n_parts; ++p)
    if (ranges[p + 1] <= ranges[p]) return "part ranges must be strictly increasing";
  L = LocalMesh();
  L.part = part;
  L.n_parts = n_parts;
  L.own_begin = ranges[part];
  L.own_end = ranges[part + 1];
  L.n_own = L.own_end - L.own_begin;
  std::vector<int32_t> beams, quads;
  part_elements(n_nodes, n_beams, beam_conn, n_quads, quad_conn, L.own_begin, L.own_end, beams, quads);
  std::vector<int32_t> halo = halo_nodes(ranges, n_parts, part, beam_conn, quad_conn, beams, quads);
  L.node_gid.resize((size_t)L.n_own + halo.size());
  for (int32_t i = 0; i < L.n_own; ++i) L.node_gid[i] = L.own_begin + i;
  for (size_t i = 0; i < halo.size(); ++i) L.node_gid[L.n_own + i] = halo[i];
  auto local_id = [&](int32_t g) -> int32_t {
    if (g >= L.own_begin && g < L.own_end) return g - L.own_begin;
    auto it = std::lower_bound(halo.begin(), halo.end(), g);
    return L.n_own + (int32_t)(it - halo.begin());
  };
  L.beam_gid = beams;
  L.quad_gid = quads;
  L.beam_conn.resize(2 * beams.size());
  for (size_t k = 0; k < beams.size(); ++k)
    for (int i = 0; i < 2; ++i) L.beam_conn[2 * k + i] = local_id(beam_conn[2 * beams[k] + i]);
  L.quad_conn.resize(4 * quads.size());
  for (size_t k = 0; k < quads.size(); ++k) {
    for (int i = 0; i < 4; ++i) L.quad_conn[4 * k + i] = local_id(quad_conn[4 * (int64_t)quads[k] + i]);
    const int32_t first = quad_conn[4 * (int64_t)quads[k]];
    if (first >= L.own_begin && first < L.own_end) L.own_quad_local.push_back((int32_t)k);
  }
  // receive plan: my halo grouped by owner (already sorted by gid -> by owner)
  size_t i = 0;
  while (i < halo.size()) {
    const int32_t own = owner_of(ranges, n_parts, halo[i]);
    size_t j = i;
    while (j < halo.size() && owner_of(ranges, n_parts, halo[j]) == own) ++j;
    NeighborPlan nb;
    nb.part = own;
    nb.recv_offset = (int32_t)i;
    nb.recv_count = (int32_t)(j - i);
    L.nbrs.push_back(nb);
    i = j;
  }
  // send plan: for every other part q, the nodes of my range in q's halo (q's halo order)
  for (int32_t q = 0; q < n_parts; ++q) {
    if (q == part) continue;
    std::vector<int32_t> qb, qq;
    part_elements(n_nodes, n_beams, beam_conn, n_quads, quad_conn, ranges[q], ranges[q + 1], qb, qq);
    std::vector<int32_t> qh = halo_nodes(ranges, n_parts, q, beam_conn, quad_conn, qb, qq);
    std::vector<int32_t> send;
    for (int32_t g : qh)
      if (g >= L.own_begin && g < L.own_end) send.push_back(g - L.own_begin);
    if (send.empty()) continue;
    auto it = std::find_if(L.nbrs.begin(), L.nbrs.end(), [&](const NeighborPlan& n) { return n.part == q; });
    if (it == L.nbrs.end()) {
      NeighborPlan nb;
      nb.part = q;
      L.nbrs.push_back(nb);
      it = L.nbrs.end() - 1;
    }
    it->send_local = send;
  }
  std::sort(L.nbrs.begin(), L.nbrs.end(), [](const NeighborPlan& a, const NeighborPlan& b) { return a.part < b.part; });
  return std::string();
}

}  // namespace sso
