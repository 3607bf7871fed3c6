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

}  // namespace sso
