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

int qtn_internal_set_error(int code, const char* msg);

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

// ---------------------------------------------------------------------------
// Dry run and greedy slicing: restatements of the
// reference's dry_run / _assign_buckets (src/ordering.py:97-145) and
// suggest_slicing / _bucket_union (src/ordering.py:192-230) over index sets.
// ---------------------------------------------------------------------------
namespace {

struct Replay {
  // active order (fixed indices removed) and each id's position in it
  std::vector<int64_t> active;
  std::unordered_map<int64_t, int32_t> pos;
  // tensors' index sets (fixed ids removed), sorted by id
  std::vector<std::vector<int64_t>> sets;
};

int build_replay(int32_t n_tensors, const int32_t* tensor_ptr, const int64_t* tensor_idx, int32_t n_order,
                 const int64_t* order, const std::vector<int64_t>& fixed, Replay* R) {
  std::unordered_map<int64_t, char> fx;
  for (int64_t f : fixed) fx[f] = 1;
  R->active.clear();
  R->pos.clear();
  for (int32_t i = 0; i < n_order; ++i)
    if (!fx.count(order[i])) {
      if (R->pos.count(order[i])) return qtn_internal_set_error(QTN_E_INVALID, "duplicate id in the order");
      R->pos[order[i]] = (int32_t)R->active.size();
      R->active.push_back(order[i]);
    }
  R->sets.assign(n_tensors, {});
  for (int32_t t = 0; t < n_tensors; ++t) {
    auto& s = R->sets[t];
    for (int32_t j = tensor_ptr[t]; j < tensor_ptr[t + 1]; ++j)
      if (!fx.count(tensor_idx[j])) s.push_back(tensor_idx[j]);
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
  }
  return QTN_OK;
}

// The replay: widths of every active bucket, or (target_step >= 0) the union
// of that bucket's sets before its own index is removed.
void run_replay(const Replay& R, int64_t target_step, std::vector<int32_t>* widths, std::vector<int64_t>* union_out) {
  const size_t n = R.active.size();
  std::vector<std::vector<std::vector<int64_t>>> buckets(n);
  auto first_pos = [&](const std::vector<int64_t>& s) {
    int32_t best = -1;
    for (int64_t x : s) {
      auto it = R.pos.find(x);
      if (it != R.pos.end() && (best < 0 || it->second < best)) best = it->second;
    }
    return best;
  };
  for (const auto& s : R.sets) {
    const int32_t p = first_pos(s);
    if (p >= 0) buckets[p].push_back(s);   // fully open / scalar sets do no bucket work
  }
  if (widths) widths->clear();
  std::vector<int64_t> uni;
  for (size_t step = 0; step < n; ++step) {
    uni.clear();
    for (const auto& s : buckets[step]) uni.insert(uni.end(), s.begin(), s.end());
    std::sort(uni.begin(), uni.end());
    uni.erase(std::unique(uni.begin(), uni.end()), uni.end());
    if ((int64_t)step == target_step) {
      *union_out = uni;
      return;
    }
    uni.erase(std::remove(uni.begin(), uni.end(), R.active[step]), uni.end());
    if (widths) widths->push_back((int32_t)uni.size());
    const int32_t p = first_pos(uni);
    if (p >= 0) buckets[p].push_back(uni);
    std::vector<std::vector<int64_t>>().swap(buckets[step]);
  }
}

}  // namespace

extern "C" int qtn_dry_run(int32_t n_tensors, const int32_t* tensor_ptr, const int64_t* tensor_idx, int32_t n_order,
                           const int64_t* order, int32_t n_fixed, const int64_t* fixed, int32_t* widths_out,
                           int64_t* active_out, int32_t* n_out) {
  if (n_tensors < 0 || n_order < 0 || n_fixed < 0 || !n_out || (n_tensors > 0 && (!tensor_ptr || !tensor_idx)) ||
      (n_order > 0 && (!order || !widths_out || !active_out)) || (n_fixed > 0 && !fixed))
    return qtn_internal_set_error(QTN_E_INVALID, "qtn_dry_run: bad arguments");
  Replay R;
  int rc = build_replay(n_tensors, tensor_ptr, tensor_idx, n_order, order,
                        std::vector<int64_t>(fixed, fixed + n_fixed), &R);
  if (rc) return rc;
  std::vector<int32_t> w;
  run_replay(R, -1, &w, nullptr);
  for (size_t i = 0; i < w.size(); ++i) {
    widths_out[i] = w[i];
    active_out[i] = R.active[i];
  }
  *n_out = (int32_t)w.size();
  return QTN_OK;
}

extern "C" int qtn_suggest_slicing(int32_t n_tensors, const int32_t* tensor_ptr, const int64_t* tensor_idx,
                                   int32_t n_order, const int64_t* order, int32_t target_width, int32_t max_out,
                                   int64_t* sliced_out, int32_t* n_out) {
  if (target_width < 1) return qtn_internal_set_error(QTN_E_INVALID, "target_width must be >= 1");
  if (n_tensors < 0 || n_order < 0 || !n_out || (max_out > 0 && !sliced_out) ||
      (n_tensors > 0 && (!tensor_ptr || !tensor_idx)) || (n_order > 0 && !order))
    return qtn_internal_set_error(QTN_E_INVALID, "qtn_suggest_slicing: bad arguments");
  std::vector<int64_t> sliced;
  Replay R;
  std::vector<int32_t> w;
  std::vector<int64_t> uni;
  for (;;) {
    int rc = build_replay(n_tensors, tensor_ptr, tensor_idx, n_order, order, sliced, &R);
    if (rc) return rc;
    run_replay(R, -1, &w, nullptr);
    int32_t best = -1, step = 0;
    for (size_t i = 0; i < w.size(); ++i)
      if (w[i] > best) best = w[i], step = (int32_t)i;   // first maximum (np.argmax)
    if (best <= target_width) break;
    run_replay(R, step, nullptr, &uni);
    int64_t pick = R.active[step];
    for (int64_t x : uni)   // sorted ascending; sliced ids were removed from every set
      if (std::find(sliced.begin(), sliced.end(), x) == sliced.end()) {
        pick = x;
        break;
      }
    sliced.push_back(pick);
    if ((int32_t)sliced.size() > max_out) return qtn_internal_set_error(QTN_E_INVALID, "slicing exceeds max_out");
  }
  for (size_t i = 0; i < sliced.size(); ++i) sliced_out[i] = sliced[i];
  *n_out = (int32_t)sliced.size();
  return QTN_OK;
}
