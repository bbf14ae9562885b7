// planner.cpp — host-side elimination ordering for the C ABI.
//
// qtn_greedy_order restates the reference's greedy_order (src/ordering.py:26-94):
// line graph over index ids (two indices adjacent iff a tensor holds both); a
// (score, id) min-heap with lazy invalidation; eliminating v turns its
// live/open neighbours into a clique; min-fill scores (missing edges among the
// neighbours) or min-degree; only vertices whose score changed are re-pushed,
// so ties break toward the smallest index id.  The result is a deterministic
// function of the graph, identical to the reference's (golden-tested).
#include <algorithm>
#include <cstdint>
#include <functional>
#include <queue>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "qtn_b200.h"

namespace {

struct Graph {
  int n = 0;
  int words = 0;
  std::vector<uint64_t> bits;              // adjacency bitsets (n x words)
  std::vector<std::vector<int>> nbr;       // adjacency lists (kept in sync)

  bool has(int a, int b) const { return (bits[(size_t)a * words + (b >> 6)] >> (b & 63)) & 1ull; }
  void add(int a, int b) {
    uint64_t& w = bits[(size_t)a * words + (b >> 6)];
    const uint64_t m = 1ull << (b & 63);
    if (!(w & m)) {
      w |= m;
      nbr[a].push_back(b);
    }
  }
  void remove(int a, int b) {
    uint64_t& w = bits[(size_t)a * words + (b >> 6)];
    const uint64_t m = 1ull << (b & 63);
    if (w & m) {
      w &= ~m;
      auto& v = nbr[a];
      v.erase(std::find(v.begin(), v.end(), b));
    }
  }
};

int64_t fill_score(const Graph& g, int v) {
  const auto& ns = g.nbr[v];
  int64_t miss = 0;
  for (size_t i = 0; i < ns.size(); ++i)
    for (size_t j = i + 1; j < ns.size(); ++j)
      if (!g.has(ns[i], ns[j])) ++miss;
  return miss;
}

}  // namespace

extern "C" int qtn_greedy_order(int32_t n_tensors, const int32_t* tensor_ptr, const int64_t* tensor_idx,
                                int32_t n_open, const int64_t* open_idx, int32_t heuristic, int64_t* order_out,
                                int32_t* n_out) {
  if (n_tensors < 0 || !tensor_ptr || (n_tensors > 0 && !tensor_idx) || !order_out || !n_out ||
      (n_open > 0 && !open_idx) || (heuristic != 0 && heuristic != 1))
    return QTN_E_INVALID;
  // dense ids in sorted order of the original ids (so id comparisons match)
  std::vector<int64_t> ids(tensor_idx, tensor_idx + tensor_ptr[n_tensors]);
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  const int n = (int)ids.size();
  std::unordered_map<int64_t, int> dense;
  dense.reserve(ids.size() * 2);
  for (int i = 0; i < n; ++i) dense[ids[i]] = i;
  Graph g;
  g.n = n;
  g.words = (n + 63) / 64;
  g.bits.assign((size_t)n * g.words, 0ull);
  g.nbr.assign(n, {});
  for (int t = 0; t < n_tensors; ++t) {
    const int b = tensor_ptr[t], e = tensor_ptr[t + 1];
    for (int i = b; i < e; ++i)
      for (int j = b; j < e; ++j) {
        const int x = dense[tensor_idx[i]], y = dense[tensor_idx[j]];
        if (x != y) g.add(x, y);
      }
  }
  std::vector<char> open(n, 0), alive(n, 1);
  for (int i = 0; i < n_open; ++i) {
    auto it = dense.find(open_idx[i]);
    if (it != dense.end()) {
      open[it->second] = 1;
      alive[it->second] = 0;
    }
  }
  const bool minfill = heuristic == 0;
  auto score = [&](int v) -> int64_t { return minfill ? fill_score(g, v) : (int64_t)g.nbr[v].size(); };
  std::vector<int64_t> cur(n, 0);
  using Entry = std::pair<int64_t, int>;
  std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> heap;
  int n_alive = 0;
  for (int v = 0; v < n; ++v)
    if (alive[v]) {
      cur[v] = score(v);
      heap.push({cur[v], v});
      ++n_alive;
    }
  int out = 0;
  std::vector<int> nbrs, dirty_list;
  std::vector<char> dirty(n, 0);
  while (n_alive > 0) {
    int v = -1;
    while (!heap.empty()) {
      const Entry e = heap.top();
      heap.pop();
      if (alive[e.second] && cur[e.second] == e.first) {
        v = e.second;
        break;
      }
    }
    if (v < 0) return QTN_E_INVALID;   // cannot happen: every alive vertex has a live entry
    order_out[out++] = ids[v];
    alive[v] = 0;
    --n_alive;
    nbrs.clear();
    for (int w : g.nbr[v])
      if (alive[w] || open[w]) nbrs.push_back(w);
    const std::vector<int> all_nb = g.nbr[v];
    for (int w : all_nb) g.remove(w, v);
    for (int w : all_nb) g.remove(v, w);
    for (size_t i = 0; i < nbrs.size(); ++i)
      for (size_t j = i + 1; j < nbrs.size(); ++j) {
        const int a = nbrs[i], b = nbrs[j];
        if (!g.has(a, b)) {
          g.add(a, b);
          g.add(b, a);
        }
      }
    dirty_list.clear();
    auto mark = [&](int w) {
      if (!dirty[w]) {
        dirty[w] = 1;
        dirty_list.push_back(w);
      }
    };
    for (int w : nbrs) mark(w);
    if (minfill)
      for (int w : nbrs)
        for (int x : g.nbr[w]) mark(x);
    for (int w : dirty_list) {
      dirty[w] = 0;
      if (alive[w]) {
        const int64_t s2 = score(w);
        if (s2 != cur[w]) {
          cur[w] = s2;
          heap.push({s2, w});
        }
      }
    }
  }
  *n_out = out;
  return QTN_OK;
}
