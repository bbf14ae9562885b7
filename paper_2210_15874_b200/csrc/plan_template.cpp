// plan_template.cpp — the symbolic program planner in C++ (SURVEY 8(f) row 1).
//
// Restates engine.plan_template (Python, kept as the checker): replay of
// contract_network's bucket assignment (src/ordering.py:165-187) over index
// sets only, chain merging of buckets into k-sum items under the same cost
// model, and the per-item layout (tile bits, smem staging, step mask, member
// classes, kernel variant).  Every decision uses the same integer / double
// arithmetic in the same order as the Python planner, so the two produce
// identical templates (tests/test_planner_cpu.py compares them array by
// array).  Cost-model constants come from the caller (engine.py is the
// single source of truth).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <string>
#include <unordered_map>
#include <vector>

#include "qtn_b200.h"

int qtn_internal_set_error(int code, const char* msg);

namespace {

using std::vector;

struct Mem {
  int kind;           // 0 = input tensor, 1 = item (planner-internal id)
  int64_t ref;
  vector<int> set;    // positions in the active order, ascending
};

struct Item {
  vector<int> X;      // summed positions, ascending
  vector<int> R;      // result positions, ascending
  vector<Mem> mem;
  vector<int> refs;
  double cost = 0.0;
  bool dead = false;
};

inline int popc64(uint64_t x) { return __builtin_popcountll(x); }
inline int64_t align_up(int64_t n, int64_t a) { return (n + a - 1) / a * a; }
inline int64_t tensor_align(int64_t size) { return std::max<int64_t>(1, std::min<int64_t>(size, 32)); }

struct Planner {
  qtn_plan_params_t P;
  int sib = 12;

  void masks(const vector<Mem>& mem, const vector<int>& X, const vector<int>& R, vector<uint64_t>& m,
             vector<uint64_t>& sm) const {
    const int w = (int)R.size(), k = (int)X.size();
    m.assign(mem.size(), 0);
    sm.assign(mem.size(), 0);
    for (size_t i = 0; i < mem.size(); ++i)
      for (int a : mem[i].set) {
        auto it = std::lower_bound(R.begin(), R.end(), a);
        if (it != R.end() && *it == a) {
          m[i] |= 1ull << (w - 1 - (int)(it - R.begin()));
        } else {
          auto jt = std::lower_bound(X.begin(), X.end(), a);
          sm[i] |= 1ull << (k - 1 - (int)(jt - X.begin()));
        }
      }
  }

  // engine._tile_bits
  int tile_bits(int w, const vector<uint64_t>& m, const vector<uint64_t>& sm, int64_t* st_out) const {
    int L = std::min(w, P.tile_bits);
    for (;;) {
      const uint64_t low = (L >= 64) ? ~0ull : ((1ull << L) - 1);
      int64_t st = 0;
      for (size_t i = 0; i < m.size(); ++i)
        if ((m[i] & low) != low) st += ((int64_t)1 << popc64(sm[i]) << popc64(m[i] & low)) + 1;
      st += (int64_t)1 << P.kmax;
      if (st * P.elem_bytes <= P.smem_budget || L == 0) {
        // wave-aware: a smaller tile when the last wave of the persistent
        // grid would run mostly empty (engine._tile_bits)
        if (P.wave_slots > 0) {
          const int lmin = std::max(std::min(w, P.min_tile_bits), L - 2);
          int best = L;
          int64_t best_t = -1;
          for (int l = L; l >= lmin; --l) {
            const int64_t tiles = (int64_t)1 << (w - l);
            const int64_t t = (tiles + P.wave_slots - 1) / P.wave_slots * (((int64_t)1 << l) + P.wave_ov_elems);
            if (best_t < 0 || t < best_t) best = l, best_t = t;
          }
          if (best != L) {
            L = best;
            const uint64_t low2 = (1ull << L) - 1;
            st = 0;
            for (size_t i = 0; i < m.size(); ++i)
              if ((m[i] & low2) != low2) st += ((int64_t)1 << popc64(sm[i]) << popc64(m[i] & low2)) + 1;
            st += (int64_t)1 << P.kmax;
          }
        }
        if (st_out) *st_out = st;
        return L;
      }
      --L;
    }
  }

  // engine._item_cost (nm_eff < 0: every member counts 1)
  double item_cost(int w, int k, int L, const vector<int64_t>& sizes, double hop, double nm_eff = -1.0) const {
    const int64_t nm_cnt = std::max<int64_t>(1, (int64_t)sizes.size());
    int64_t ssum = 0;
    for (int64_t s : sizes) ssum += s;
    const int64_t byt = (int64_t)P.elem_bytes * (((int64_t)1 << w) + ssum);
    const int64_t tiles = (int64_t)1 << (w - L);
    const int64_t waves = (tiles + P.resident_blocks - 1) / P.resident_blocks;
    const int64_t nelem = (int64_t)1 << L;
    double per_tile;
    if (nelem >= (int64_t)P.vec * P.nt) {
      if (nm_eff < 0)
        per_tile = (double)((nelem << k) * nm_cnt) / P.block_terms_ps;
      else
        per_tile = (double)(nelem << k) * nm_eff / P.block_terms_ps;
    } else {
      const int64_t rounds = ((nelem << k) + 2 * P.nt - 1) / (2 * P.nt);
      per_tile = 1e-6 + (double)rounds * P.small_load_s;
    }
    const double a = (double)byt / P.bw_bps;
    const double b = (double)waves * per_tile;
    return hop + std::max(a, b);
  }

  // engine._cost_of
  double cost_of(const Item& it) const {
    vector<uint64_t> m, sm;
    masks(it.mem, it.X, it.R, m, sm);
    const int w = (int)it.R.size(), k = (int)it.X.size();
    vector<int64_t> sizes;
    for (const Mem& mm : it.mem) sizes.push_back((int64_t)1 << mm.set.size());
    if (w + k <= sib) return item_cost(w, k, std::min(w, P.small_tile_bits), sizes, P.hop_k2_s);
    const int L = tile_bits(w, m, sm, nullptr);
    double nm_eff = -1.0;
    if (P.cheap_member_w != 1.0 && ((int64_t)1 << L) >= (int64_t)P.vec * P.nt) {
      const uint64_t stm = step_mask(L, m);
      const uint64_t full = (1ull << L) - 1;
      int n_cheap = 0;
      for (uint64_t x : m) {
        const uint64_t lo = x & full;
        if (lo != full && (lo == 0 || (k <= 3 && (lo & stm) == 0))) ++n_cheap;
      }
      nm_eff = std::max(1.0, (double)((int)m.size() - n_cheap) + P.cheap_member_w * (double)n_cheap);
    }
    return item_cost(w, k, L, sizes, P.hop_s, nm_eff);
  }

  // engine._step_mask: maximise (invariant staged members, mask)
  uint64_t step_mask(int L, const vector<uint64_t>& m) const {
    const int lb = P.vec == 2 ? 1 : 0;
    const int n_st = L - lb - 8;
    if (n_st <= 0) return 0;
    const uint64_t full = (1ull << L) - 1;
    vector<uint64_t> staged;
    for (uint64_t x : m)
      if ((x & full) != full) staged.push_back(x & full);
    const int lo = lb + 5;
    uint64_t best = 0;
    int best_inv = -1;
    for (uint64_t s = 0; s < (1ull << (L - lo)); ++s) {
      if (popc64(s) != n_st) continue;
      const uint64_t sm = s << lo;
      int inv = 0;
      for (uint64_t x : staged)
        if ((x & sm) == 0) ++inv;
      if (inv > best_inv || (inv == best_inv && sm > best)) {
        best = sm;
        best_inv = inv;
      }
    }
    return best;
  }
};

}  // namespace

struct qtn_plan {
  vector<vector<int64_t>> arr;   // indexed by QTN_PLAN_*
  vector<int64_t> fixed_ids;
  int64_t scalars[8] = {};
};

extern "C" {

int qtn_plan_build(int32_t n_tensors, const int32_t* tensor_ptr, const int64_t* tensor_idx, int32_t n_order,
                   const int64_t* order, int32_t n_fixed, const int64_t* fixed, const qtn_plan_params_t* params,
                   qtn_plan_t** out) {
  if (!out || !params || (n_tensors > 0 && !tensor_ptr) || n_tensors < 0 || n_order < 0 || n_fixed < 0)
    return qtn_internal_set_error(QTN_E_INVALID, "null argument");
  Planner PL;
  PL.P = *params;
  PL.sib = params->small_iter_bits;
  std::unordered_map<int64_t, int> fixpos;
  for (int i = 0; i < n_fixed; ++i) fixpos.emplace(fixed[i], i);
  // active order and positions
  std::unordered_map<int64_t, int> pos;
  vector<int64_t> act;
  for (int i = 0; i < n_order; ++i)
    if (!fixpos.count(order[i]) && !pos.count(order[i])) {
      pos.emplace(order[i], (int)act.size());
      act.push_back(order[i]);
    }
  const int na = (int)act.size();

  qtn_plan* R = new qtn_plan();
  R->arr.assign(QTN_PLAN_N_ARRAYS, {});
  for (int i = 0; i < n_fixed; ++i) R->fixed_ids.push_back(fixed[i]);
  auto& in_off = R->arr[QTN_PLAN_IN_OFF];
  auto& gdst = R->arr[QTN_PLAN_GDST];
  auto& gsrc = R->arr[QTN_PLAN_GSRC];
  auto& gfix = R->arr[QTN_PLAN_GFIX];   // n_fixed rows of n_canon
  vector<vector<int64_t>> gfix_rows(n_fixed);

  // ---- inputs: canonical layout and gather maps ----
  int64_t cur = 0, n_raw = 0;
  vector<vector<int>> sets(n_tensors);
  in_off.assign(n_tensors, -1);
  for (int t = 0; t < n_tensors; ++t) {
    const int64_t* idx = tensor_idx + tensor_ptr[t];
    const int r0 = tensor_ptr[t + 1] - tensor_ptr[t];
    vector<int> canon;       // positions
    vector<int> axis;        // own axis of each canonical position
    vector<int64_t> missing;
    for (int a = 0; a < r0; ++a) {
      if (fixpos.count(idx[a])) continue;
      auto it = pos.find(idx[a]);
      if (it == pos.end()) {
        missing.push_back(idx[a]);
        continue;
      }
      canon.push_back(it->second);
      axis.push_back(a);
    }
    if (!missing.empty()) {
      std::sort(missing.begin(), missing.end());
      missing.erase(std::unique(missing.begin(), missing.end()), missing.end());
      std::string msg = "order is missing indices: [";
      for (size_t q = 0; q < missing.size(); ++q) msg += (q ? ", " : "") + std::to_string(missing[q]);
      msg += "]";
      delete R;
      return qtn_internal_set_error(QTN_E_INVALID, msg.c_str());
    }
    vector<int> ordp(canon.size());
    for (size_t q = 0; q < ordp.size(); ++q) ordp[q] = (int)q;
    std::sort(ordp.begin(), ordp.end(), [&](int a, int b) { return canon[a] < canon[b]; });
    const int r = (int)canon.size();
    const int64_t size = (int64_t)1 << r;
    cur = align_up(cur, tensor_align(size));
    in_off[t] = cur;
    vector<int64_t> wts(r);
    for (int p = 0; p < r; ++p) wts[p] = (int64_t)1 << (r0 - 1 - axis[ordp[p]]);
    for (int64_t k = 0; k < size; ++k) {
      int64_t s = 0;
      for (int p = 0; p < r; ++p)
        if ((k >> (r - 1 - p)) & 1) s += wts[p];
      gdst.push_back(cur + k);
      gsrc.push_back(n_raw + s);
    }
    for (int f = 0; f < n_fixed; ++f) {
      int64_t wgt = 0;
      for (int a = 0; a < r0; ++a)
        if (idx[a] == fixed[f]) wgt = (int64_t)1 << (r0 - 1 - a);
      gfix_rows[f].insert(gfix_rows[f].end(), size, wgt);
    }
    cur += size;
    n_raw += (int64_t)1 << r0;
    vector<int> st;
    for (int p = 0; p < r; ++p) st.push_back(canon[ordp[p]]);
    sets[t] = st;   // ascending positions
  }
  const int64_t n_in = align_up(cur, 32);
  for (auto& row : gfix_rows) gfix.insert(gfix.end(), row.begin(), row.end());

  // ---- reference bucket replay ----
  struct RefB {
    int x;
    vector<Mem> mem;
    vector<int> R;
  };
  vector<vector<Mem>> pending(na);
  vector<std::pair<int, int64_t>> fin;   // (kind, ref)
  for (int t = 0; t < n_tensors; ++t) {
    if (sets[t].empty())
      fin.push_back({0, t});
    else
      pending[sets[t][0]].push_back({0, t, sets[t]});
  }
  vector<RefB> refs;
  for (int x = 0; x < na; ++x) {
    vector<Mem> mem = std::move(pending[x]);
    if (mem.empty()) continue;
    vector<int> uni;
    for (const Mem& m : mem) uni.insert(uni.end(), m.set.begin(), m.set.end());
    std::sort(uni.begin(), uni.end());
    uni.erase(std::unique(uni.begin(), uni.end()), uni.end());
    uni.erase(std::remove(uni.begin(), uni.end(), x), uni.end());
    if ((int)uni.size() > QTN_MAX_WIDTH) {
      delete R;
      char buf[96];
      snprintf(buf, sizeof(buf), "bucket width %d exceeds %d", (int)uni.size(), QTN_MAX_WIDTH);
      return qtn_internal_set_error(QTN_E_INVALID, buf);
    }
    const int b = (int)refs.size();
    refs.push_back({x, mem, uni});
    if (!uni.empty())
      pending[uni[0]].push_back({1, b, uni});
    else
      fin.push_back({1, b});
  }

  // ---- merge chains into items ----
  vector<Item> items;
  vector<int> item_of;
  for (int b = 0; b < (int)refs.size(); ++b) {
    Item it;
    it.X = {refs[b].x};
    it.R = refs[b].R;
    it.refs = {b};
    for (const Mem& m : refs[b].mem) it.mem.push_back({m.kind, m.kind == 1 ? item_of[m.ref] : m.ref, m.set});
    it.cost = PL.cost_of(it);
    bool changed = params->merge != 0;
    while (changed) {
      changed = false;
      for (size_t mi = 0; mi < it.mem.size(); ++mi) {
        const Mem& mm = it.mem[mi];
        if (mm.kind != 1 || items[mm.ref].dead) continue;
        const Item& p = items[mm.ref];
        vector<int> X2 = it.X;
        X2.insert(X2.end(), p.X.begin(), p.X.end());
        std::sort(X2.begin(), X2.end());
        X2.erase(std::unique(X2.begin(), X2.end()), X2.end());
        const size_t nmem2 = it.mem.size() - 1 + p.mem.size();
        if ((int)X2.size() > params->kmax || (int)nmem2 > params->max_members) continue;
        Item cand;
        cand.X = X2;
        cand.R = it.R;
        cand.mem.assign(it.mem.begin(), it.mem.begin() + mi);
        cand.mem.insert(cand.mem.end(), p.mem.begin(), p.mem.end());
        cand.mem.insert(cand.mem.end(), it.mem.begin() + mi + 1, it.mem.end());
        const int w = (int)it.R.size();
        if (w + (int)X2.size() > PL.sib) {
          vector<uint64_t> m, sm;
          PL.masks(cand.mem, X2, it.R, m, sm);
          const int L = PL.tile_bits(w, m, sm, nullptr);
          if (L < std::min(w, params->min_tile_bits)) continue;
        }
        if (w + (int)X2.size() > PL.sib && (int)X2.size() > params->kmax_large) continue;
        const double c2 = PL.cost_of(cand);
        if (c2 >= it.cost + p.cost) continue;
        const int64_t pr = mm.ref;
        vector<int> refs2 = items[pr].refs;
        refs2.insert(refs2.end(), it.refs.begin(), it.refs.end());
        it.X = X2;
        it.mem = std::move(cand.mem);
        it.cost = c2;
        it.refs = std::move(refs2);
        items[pr].dead = true;
        changed = true;
        break;
      }
    }
    item_of.push_back((int)items.size());
    items.push_back(std::move(it));
  }

  // ---- compact, layout ----
  vector<int> renum(items.size(), -1);
  int nlive = 0;
  for (size_t i = 0; i < items.size(); ++i)
    if (!items[i].dead) renum[i] = nlive++;
  auto& W = R->arr[QTN_PLAN_W];
  auto& K = R->arr[QTN_PLAN_K];
  auto& Ls = R->arr[QTN_PLAN_L];
  auto& lev = R->arr[QTN_PLAN_LEVEL];
  auto& outo = R->arr[QTN_PLAN_OUT_OFF];
  auto& mptr = R->arr[QTN_PLAN_MEM_PTR];
  auto& mkind = R->arr[QTN_PLAN_MEM_KIND];
  auto& mref = R->arr[QTN_PLAN_MEM_REF];
  auto& mmask = R->arr[QTN_PLAN_MEM_MASK];
  auto& msmask = R->arr[QTN_PLAN_MEM_SMASK];
  auto& smem = R->arr[QTN_PLAN_SMEM];
  auto& stm = R->arr[QTN_PLAN_STMASK];
  auto& mcls = R->arr[QTN_PLAN_MEM_CLS];
  auto& var = R->arr[QTN_PLAN_VARIANT];
  auto& ref_item = R->arr[QTN_PLAN_REF_ITEM];
  auto& ref_last = R->arr[QTN_PLAN_REF_LAST];
  ref_item.assign(refs.size(), 0);
  ref_last.assign(refs.size(), 0);
  mptr.push_back(0);
  int64_t inter = 0;
  const int64_t vecnt = (int64_t)params->vec * params->nt;
  for (size_t old = 0; old < items.size(); ++old) {
    const Item& it = items[old];
    if (it.dead) continue;
    const int nw = renum[old];
    const int w = (int)it.R.size(), k = (int)it.X.size();
    vector<uint64_t> m, sm;
    PL.masks(it.mem, it.X, it.R, m, sm);
    int L;
    int64_t st = 0;
    if (w + k <= PL.sib)
      L = std::min(w, params->small_tile_bits);
    else
      L = PL.tile_bits(w, m, sm, &st);
    int64_t lv = 0;
    for (size_t j = 0; j < it.mem.size(); ++j) {
      int64_t rr = it.mem[j].ref;
      if (it.mem[j].kind == 1) {
        rr = renum[rr];
        lv = std::max(lv, lev[rr] + 1);
      }
      mkind.push_back(it.mem[j].kind);
      mref.push_back(rr);
      mmask.push_back((int64_t)m[j]);
      msmask.push_back((int64_t)sm[j]);
    }
    mptr.push_back((int64_t)mkind.size());
    const int64_t size = (int64_t)1 << w;
    inter = align_up(inter, tensor_align(size));
    W.push_back(w);
    K.push_back(k);
    Ls.push_back(L);
    lev.push_back(lv);
    outo.push_back(inter);
    smem.push_back(st);
    const uint64_t sm_ = ((int64_t)1 << L) >= vecnt ? PL.step_mask(L, m) : 0;
    stm.push_back((int64_t)sm_);
    // member classes (engine.member_classes) and variant (engine.kernel_variant)
    const uint64_t full = (1ull << L) - 1;
    int nv = 0, nst = 0, nb0 = 0;
    for (size_t j = 0; j < m.size(); ++j) {
      const uint64_t lo = m[j] & full;
      int c;
      if (lo == full)
        c = QTN_CLS_STREAMED;
      else if (lo == 0)
        c = QTN_CLS_UNIFORM;
      else if (k <= 3 && (lo & sm_) == 0)
        c = QTN_CLS_INVARIANT;
      else
        c = QTN_CLS_VARYING;
      mcls.push_back(c);
      if (c == QTN_CLS_VARYING) {
        ++nv;
        if (params->vec == 2 && (m[j] & 1)) ++nb0;
      }
      if (c == QTN_CLS_STREAMED) ++nst;
    }
    int64_t v;
    if (((int64_t)1 << L) < vecnt)
      v = -2;   // VARIANT_SMALL
    else if (k <= 3 && nv <= 4 && nst <= 1)
      v = k | (nv << 4) | (nst << 8) | (nb0 << 12);
    else
      v = QTN_VARIANT_GENERIC;
    var.push_back(v);
    inter += size;
    for (int r_ : it.refs) ref_item[r_] = nw;
    ref_last[it.refs.back()] = 1;
  }
  auto& ref_w = R->arr[QTN_PLAN_REF_W];
  auto& ref_elems = R->arr[QTN_PLAN_REF_ELEMS];
  auto& bidx = R->arr[QTN_PLAN_BUCKET_INDEX];
  int64_t maxw = 0;
  for (const RefB& rb : refs) {
    ref_w.push_back((int64_t)rb.R.size());
    int64_t e = (int64_t)1 << rb.R.size();
    for (const Mem& mm : rb.mem) e += (int64_t)1 << mm.set.size();
    ref_elems.push_back(e);
    bidx.push_back(act[rb.x]);
    maxw = std::max<int64_t>(maxw, (int64_t)rb.R.size());
  }
  auto& fk = R->arr[QTN_PLAN_FIN_KIND];
  auto& fr = R->arr[QTN_PLAN_FIN_REF];
  for (auto& f : fin) {
    fk.push_back(f.first);
    fr.push_back(f.first == 1 ? ref_item[f.second] : f.second);
  }
  R->scalars[0] = n_in;
  R->scalars[1] = align_up(inter, 32);
  R->scalars[2] = n_raw;
  R->scalars[3] = maxw;
  *out = R;
  return QTN_OK;
}

int qtn_plan_scalars(const qtn_plan_t* p, int64_t* s) {
  if (!p || !s) return qtn_internal_set_error(QTN_E_INVALID, "null plan");
  for (int i = 0; i < 4; ++i) s[i] = p->scalars[i];
  return QTN_OK;
}

int qtn_plan_array_len(const qtn_plan_t* p, int32_t id, int64_t* len) {
  if (!p || !len || id < 0 || id >= QTN_PLAN_N_ARRAYS) return qtn_internal_set_error(QTN_E_INVALID, "bad plan array");
  *len = (int64_t)p->arr[id].size();
  return QTN_OK;
}

int qtn_plan_array(const qtn_plan_t* p, int32_t id, int64_t* dst) {
  if (!p || id < 0 || id >= QTN_PLAN_N_ARRAYS) return qtn_internal_set_error(QTN_E_INVALID, "bad plan array");
  const auto& a = p->arr[id];
  if (!a.empty()) {
    if (!dst) return qtn_internal_set_error(QTN_E_INVALID, "null destination");
    std::copy(a.begin(), a.end(), dst);
  }
  return QTN_OK;
}

int qtn_plan_destroy(qtn_plan_t* p) {
  delete p;
  return QTN_OK;
}

}  // extern "C"
