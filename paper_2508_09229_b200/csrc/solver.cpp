// Host min-cost flow for solve_exact.
//
// The ILP of Eq. (1) is a transportation problem whose constraint matrix is a network matrix
// (SPEC.md:302), so an integral min-cost max-flow optimum is an ILP optimum.  Network:
//   source -> item(l,e)            cap 1,        cost 0
//   item(l,e) -> slot(l,s)         cap 1,        cost w[l,e,s]         (full form, p == NULL)
//   slot(l,s) -> server(s)         cap c_layer,  cost 0
//   server(s) -> sink              cap c_exp,    cost 0
// Class compression (p != NULL): when w[l,e,s] depends on s only through p[l,s] (always true
// for build_instance output, w = f * p), all slots of one layer with equal p are
// interchangeable for every item, so item(l,e) -> class(l,v) (cap 1, cost w[l,e,s in class])
// and class(l,v) -> server(s) (cap c_layer) for each s with p[l,s] = v is an equivalent network
// with ~S/|classes| times fewer arcs.  The flow on class->server arcs is then distributed to
// the class's items in ascending (e, s) order.
//
// Algorithm: primal-dual successive shortest paths.  Dijkstra on reduced costs (binary heap,
// potentials keep them >= 0), then a Dinic blocking flow on the zero-reduced-cost residual
// subgraph, repeated until the flow reaches L*E or the sink becomes unreachable.
#include <cstdint>
#include <cstring>
#include <vector>
#include <queue>
#include <algorithm>
#include <atomic>
#include <thread>
#include <limits>
#include "../../include/moeplace_cuda.h"

namespace {

struct MCF {
  struct Arc {
    int to;
    int cap;
    int64_t cost;
  };
  int n;
  std::vector<int> head_start;  // CSR after finalize
  std::vector<int> adj;         // arc ids per node (CSR)
  std::vector<Arc> arcs;        // arc i and i^1 are a residual pair
  std::vector<std::vector<int>> tmp_adj;

  explicit MCF(int n_) : n(n_), tmp_adj(n_) {}

  int add(int u, int v, int cap, int64_t cost) {
    const int id = (int)arcs.size();
    arcs.push_back({v, cap, cost});
    arcs.push_back({u, 0, -cost});
    tmp_adj[u].push_back(id);
    tmp_adj[v].push_back(id + 1);
    return id;
  }
  void finalize() {
    head_start.assign(n + 1, 0);
    for (int u = 0; u < n; ++u) head_start[u + 1] = head_start[u] + (int)tmp_adj[u].size();
    adj.resize(head_start[n]);
    for (int u = 0; u < n; ++u) std::copy(tmp_adj[u].begin(), tmp_adj[u].end(), adj.begin() + head_start[u]);
    tmp_adj.clear();
    tmp_adj.shrink_to_fit();
  }
  int from(int id) const { return arcs[id ^ 1].to; }

  // returns total flow; cost accumulated in *cost
  int64_t run(int s, int t, int64_t need, int64_t* total_cost) {
    const int64_t INF = std::numeric_limits<int64_t>::max() / 4;
    std::vector<int64_t> pot(n, 0), dist(n);
    std::vector<int> level(n), it(n);
    std::vector<char> done(n);
    int64_t flow = 0, cost = 0;
    using QE = std::pair<int64_t, int>;
    while (flow < need) {
      // Dijkstra on reduced costs
      std::fill(dist.begin(), dist.end(), INF);
      std::fill(done.begin(), done.end(), 0);
      std::priority_queue<QE, std::vector<QE>, std::greater<QE>> pq;
      dist[s] = 0;
      pq.push({0, s});
      while (!pq.empty()) {
        auto [d, u] = pq.top();
        pq.pop();
        if (done[u]) continue;
        done[u] = 1;
        if (u == t) break;
        for (int k = head_start[u]; k < head_start[u + 1]; ++k) {
          const Arc& a = arcs[adj[k]];
          if (a.cap <= 0) continue;
          const int64_t nd = d + a.cost + pot[u] - pot[a.to];
          if (nd < dist[a.to]) {
            dist[a.to] = nd;
            pq.push({nd, a.to});
          }
        }
      }
      if (dist[t] >= INF) break;
      const int64_t dt = dist[t];
      for (int v = 0; v < n; ++v) pot[v] += std::min(dist[v], dt);
      // blocking flows on the admissible (zero reduced cost) subgraph
      while (flow < need) {
        // BFS levels over admissible arcs
        std::fill(level.begin(), level.end(), -1);
        std::vector<int> q;
        q.reserve(n);
        q.push_back(s);
        level[s] = 0;
        for (size_t qi = 0; qi < q.size(); ++qi) {
          const int u = q[qi];
          for (int k = head_start[u]; k < head_start[u + 1]; ++k) {
            const Arc& a = arcs[adj[k]];
            if (a.cap > 0 && level[a.to] < 0 && a.cost + pot[u] - pot[a.to] == 0) {
              level[a.to] = level[u] + 1;
              q.push_back(a.to);
            }
          }
        }
        if (level[t] < 0) break;
        for (int v = 0; v < n; ++v) it[v] = head_start[v];
        // iterative DFS augmenting unit (or bottleneck) paths
        std::vector<int> path;  // arc ids
        while (flow < need) {
          path.clear();
          int u = s;
          bool found = false;
          while (true) {
            if (u == t) { found = true; break; }
            bool advanced = false;
            for (int& k = it[u]; k < head_start[u + 1]; ++k) {
              const int id = adj[k];
              const Arc& a = arcs[id];
              if (a.cap > 0 && level[a.to] == level[u] + 1 && a.cost + pot[u] - pot[a.to] == 0) {
                path.push_back(id);
                u = a.to;
                advanced = true;
                break;
              }
            }
            if (!advanced) {
              if (u == s) break;
              level[u] = -1;  // dead end
              const int id = path.back();
              path.pop_back();
              u = from(id);
              ++it[u];
            }
          }
          if (!found) break;
          int64_t b = need - flow;
          for (int id : path) b = std::min<int64_t>(b, arcs[id].cap);
          for (int id : path) {
            arcs[id].cap -= (int)b;
            arcs[id ^ 1].cap += (int)b;
            cost += b * arcs[id].cost;
          }
          flow += b;
        }
      }
    }
    *total_cost = cost;
    return flow;
  }
};

}  // namespace

// Min-cost flow over layers [l0, l1) (indices into the full w / p / assign arrays).
static int solve_layers(const int64_t* w, const uint8_t* p, int l0, int l1, int E, int S, int c_layer, int c_exp,
                        bool compress, const std::vector<int>* cls_of_all, const std::vector<int>* cls_rep_all,
                        int32_t* assign_out, int64_t* objective_out, int64_t* flow_out) {
  // node numbering
  const int L = l1 - l0;
  const int64_t LE = (int64_t)L * E;
  w += (int64_t)l0 * E * S;
  if (p) p += (int64_t)l0 * S;
  assign_out += (int64_t)l0 * E;
  const std::vector<int>* cls_of = cls_of_all + l0;
  const std::vector<int>* cls_rep = cls_rep_all + l0;
  const int src = 0;
  const int item0 = 1;
  std::vector<int> mid0(L + 1);  // first class/slot node of layer l
  mid0[0] = item0 + (int)LE;
  for (int l = 0; l < L; ++l) mid0[l + 1] = mid0[l] + (compress ? (int)cls_rep[l].size() : S);
  const int srv0 = mid0[L];
  const int sink = srv0 + S;
  MCF g(sink + 1);

  std::vector<int> item_arc0((size_t)LE);  // first item->mid arc id
  for (int64_t i = 0; i < LE; ++i) g.add(src, item0 + (int)i, 1, 0);
  for (int l = 0; l < L; ++l)
    for (int e = 0; e < E; ++e) {
      const int64_t i = (int64_t)l * E + e;
      const int64_t* row = w + i * S;
      item_arc0[i] = (int)g.arcs.size();
      if (compress) {
        for (size_t c = 0; c < cls_rep[l].size(); ++c) g.add(item0 + (int)i, mid0[l] + (int)c, 1, row[cls_rep[l][c]]);
      } else {
        for (int s = 0; s < S; ++s) g.add(item0 + (int)i, mid0[l] + s, 1, row[s]);
      }
    }
  std::vector<int> mid_arc0(L);  // first mid->server arc id per layer
  for (int l = 0; l < L; ++l) {
    mid_arc0[l] = (int)g.arcs.size();
    for (int s = 0; s < S; ++s) {
      const int m = compress ? mid0[l] + cls_of[l][s] : mid0[l] + s;
      g.add(m, srv0 + s, c_layer, 0);
    }
  }
  for (int s = 0; s < S; ++s) g.add(srv0 + s, sink, c_exp, 0);
  g.finalize();

  int64_t cost = 0;
  const int64_t flow = g.run(src, sink, LE, &cost);
  *flow_out += flow;
  *objective_out += cost;
  if (flow < LE) return MP_INFEASIBLE;

  // read back the assignment
  for (int l = 0; l < L; ++l) {
    const int nmid = compress ? (int)cls_rep[l].size() : S;
    // per class/slot: items routed there (ascending e), and server units (ascending s)
    std::vector<std::vector<int>> items(nmid), units(nmid);
    for (int e = 0; e < E; ++e) {
      const int64_t i = (int64_t)l * E + e;
      for (int c = 0; c < nmid; ++c) {
        const int id = item_arc0[i] + 2 * c;
        if (g.arcs[id].cap == 0) { items[c].push_back(e); break; }
      }
    }
    for (int s = 0; s < S; ++s) {
      const int id = mid_arc0[l] + 2 * s;
      const int used = g.arcs[id ^ 1].cap;  // flow on the arc
      const int m = compress ? cls_of[l][s] : s;
      for (int k = 0; k < used; ++k) units[m].push_back(s);
    }
    for (int c = 0; c < nmid; ++c) {
      if (items[c].size() != units[c].size()) return MP_ERR_ARG;  // cannot happen (conservation)
      for (size_t k = 0; k < items[c].size(); ++k) assign_out[(int64_t)l * E + items[c][k]] = units[c][k];
    }
  }
  return MP_OK;
}

extern "C" int mp_solve_mcf(const int64_t* w, const uint8_t* p, int L, int E, int S, int c_layer, int c_exp,
                            int32_t* assign_out, int64_t* objective_out, int64_t* flow_out) {
  if (!w || !assign_out || L <= 0 || E <= 0 || S <= 0 || c_layer <= 0 || c_exp <= 0) return MP_ERR_ARG;
  const int64_t LE = (int64_t)L * E;
  for (int64_t i = 0; i < LE * S; ++i)
    if (w[i] < 0) return MP_ERR_ARG;

  // class compression is exact only if w depends on s through p alone
  bool compress = p != nullptr;
  std::vector<std::vector<int>> cls_of(L);     // per layer: class id per device
  std::vector<std::vector<int>> cls_rep(L);    // per layer: representative device per class
  if (compress) {
    for (int l = 0; l < L; ++l) {
      std::vector<int> id_of_val(256, -1);
      cls_of[l].resize(S);
      for (int s = 0; s < S; ++s) {
        const int v = p[(int64_t)l * S + s];
        if (id_of_val[v] < 0) { id_of_val[v] = (int)cls_rep[l].size(); cls_rep[l].push_back(s); }
        cls_of[l][s] = id_of_val[v];
      }
    }
    for (int l = 0; l < L && compress; ++l)
      for (int e = 0; e < E && compress; ++e) {
        const int64_t* row = w + ((int64_t)l * E + e) * S;
        for (int s = 0; s < S; ++s)
          if (row[s] != row[cls_rep[l][cls_of[l][s]]]) { compress = false; break; }
      }
  }

  // Decoupled layers: when L * c_layer <= c_exp the per-device total can never exceed c_exp (each
  // layer puts at most c_layer experts on a device), so the c_exp arcs carry no constraint and
  // the problem splits into L independent per-layer flows -- same optimum, each a network of
  // E items and a handful of classes (all BASELINE configs; 125 s -> well under a second for
  // four R1 topologies).  Otherwise one network over all layers.
  int64_t cost = 0, flow = 0;
  int rc = MP_OK;
  if ((int64_t)L * c_layer <= (int64_t)c_exp) {
    // independent layers on host threads (each layer's flow is deterministic; rows are disjoint)
    const int nt = (int)std::max(1u, std::min<unsigned>((unsigned)L, std::min(16u, std::thread::hardware_concurrency())));
    std::atomic<int> next(0);
    std::vector<int64_t> t_cost(nt, 0), t_flow(nt, 0);
    std::vector<int> t_rc(nt, MP_OK);
    auto work = [&](int t) {
      for (int l = next++; l < L; l = next++) {
        const int r = solve_layers(w, p, l, l + 1, E, S, c_layer, c_exp, compress, cls_of.data(), cls_rep.data(),
                                   assign_out, &t_cost[t], &t_flow[t]);
        if (r != MP_OK) t_rc[t] = r;
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (int t = 0; t < nt; ++t) {
      cost += t_cost[t];
      flow += t_flow[t];
      if (t_rc[t] != MP_OK) rc = t_rc[t];
    }
  } else {
    rc = solve_layers(w, p, 0, L, E, S, c_layer, c_exp, compress, cls_of.data(), cls_rep.data(), assign_out, &cost,
                      &flow);
  }
  if (flow_out) *flow_out = flow;
  if (objective_out) *objective_out = cost;
  return rc;
}
