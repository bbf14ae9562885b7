// bucket_expand.cu — K4: the expansion-item kernel (one dominant member).
//
// Same contraction as the reference's fast_kernel (src/tensor_core.py:148-164)
// for one program item: out[r] = sum_s prod_i m_i(r, s) over the item's
// summed bits s (one bucket index, or a merged chain of up to 3).  K4 takes
// the items whose result is an EXPANSION of one dominant member B: B carries
// all but |E| <= 4 of the w result bits ("expansion bits" E), every other
// member is small inside a tile.  K1/K3 stage B's tile slice through shared
// memory and re-read it once per result (2^k x 2^|E| reads of every staged
// element); K4 reads B straight into registers instead and keeps it there for
// all 2^|E| results that share it:
//
//   tile   = 8 "thread bits" TB (B's lowest result bits: lanes read B
//            contiguously) + the expansion bits E; the other result bits H
//            select the tile (persistent grid over 2^|H| tiles)
//   F      = the product of all members except B over the tile's F bits (the
//            result bits in TB u E that any other member carries) and s:
//            2^(|F|+k) entries in shared memory, gathered from L2.  F depends
//            on the tile only through the H bits other members carry; those
//            are the HIGH bits of the tile id and every block walks a
//            contiguous run of tile ids, so F is rebuilt only when they change
//            (typically once per block)
//   thread = one B coordinate: loads B(s) for the 2^k values of s once, then
//            out[r(e)] = sum_s B(s) * F[f(e), s] for its 2^|E| results
//
// Bytes moved are the algorithmic ones (B once, every result once, the small
// members from L2); per result the inner loop is 2^k complex FMAs and one
// 2^k-wide shared-memory read.  Every index map is GF(2)-linear in the bits,
// so offsets are sums of per-bit strides (6-bit look-up tables for F).
#include "qtn_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "k4_plan.h"

namespace qtn_k4 {

// complex64 variants are compiled for >= 4 resident blocks (<= 64 registers:
// cfg-2 0.2395 -> 0.2346 ms, the default heuristic picked 32 registers with
// spills); complex128 keeps the default (4 blocks measured 1.3 % slower)
#ifndef K4_PF
#define K4_PF 0
#endif
#ifndef K4_C64_MINB
#define K4_C64_MINB 4
#endif

template <typename R, int K, int NE, int RB>
__device__ __forceinline__ void k4_body(const Plan& P);

template <typename R, int K, int NE, int RB>
__global__ void __launch_bounds__(NT, RB == 2 ? 3 : K4_C64_MINB) k4_kernel_c64(const __grid_constant__ Plan P) {
  k4_body<R, K, NE, RB>(P);
}
template <typename R, int K, int NE, int RB>
__global__ void __launch_bounds__(NT) k4_kernel_c128(const __grid_constant__ Plan P) {
  k4_body<R, K, NE, RB>(P);
}

// RB = 2: each thread also owns the B coordinate one "replica bit" over (a B
// bit no other member carries): both share every product-table row, so each
// row read from shared memory serves two results.
template <typename R, int K, int NE, int RB>
__device__ __forceinline__ void k4_body(const Plan& P) {
  using T = typename Cx<R>::T;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int NS = 1 << K;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* F = reinterpret_cast<T*>(smem_raw);
  const int nfe = 1 << (P.nF + K);                  // F entries
  uint32_t* LUT = reinterpret_cast<uint32_t*>(smem_raw + sizeof(T) * nfe);   // [member][lo 64 | hi 64]
  __shared__ int64_t sbase[MAXM + 1];
  const int tid = threadIdx.x;
  const int nm = P.nm;
  const int nlo = P.nF + K < 6 ? P.nF + K : 6;
  // F-entry offset tables (tile independent)
  for (int x = tid; x < nm * 128; x += NT) {
    const int j = x >> 7, y = x & 63, hi = (x >> 6) & 1;
    uint32_t o = 0;
    if (j != P.iB)
      for (int b = 0; b < 6; ++b) {
        const int q = hi ? nlo + b : b;
        if (((y >> b) & 1) && (hi ? q < P.nF + K : b < nlo)) o += P.fs[j][q];
      }
    LUT[x] = o;
  }
  // this thread's B coordinate
  int64_t boff = 0;
  int32_t ob = 0, fb = 0;
#pragma unroll
  for (int b = 0; b < TBB; ++b)
    if ((tid >> b) & 1) {
      boff += P.btb[b];
      ob += P.otb[b];
      fb += P.ftb[b];
    }
  // expansion bits: the low NEL unrolled (offset tables in registers), the
  // high NEH walked by a rolled loop
  constexpr int NEL = NE < 4 ? NE : 4;
  constexpr int NEH = NE - NEL;
  constexpr int NEVL = 1 << NEL;
  int32_t oe[NEVL], fe[NEVL];
#pragma unroll
  for (int e = 0; e < NEVL; ++e) {
    int32_t o = 0, f = 0;
#pragma unroll
    for (int b = 0; b < NEL; ++b)
      if ((e >> b) & 1) {
        o += P.oe[b];
        f += P.fe[b];
      }
    oe[e] = o;
    fe[e] = (fb + f) << K;
  }
  int64_t soffB[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    int64_t o = 0;
#pragma unroll
    for (int b = 0; b < K; ++b)
      if ((s >> b) & 1) o += P.bs[b];
    soffB[s] = o;
  }
  // contiguous run of tile ids per block
  const int64_t per = (P.n_tiles + gridDim.x - 1) / gridDim.x;
  int64_t h = (int64_t)blockIdx.x * per;
  const int64_t h_end = h + per < P.n_tiles ? h + per : P.n_tiles;
  __syncthreads();
  if (h >= h_end) return;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  unsigned long long t_start = 0;
  if (P.timing && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const T* Bm = reinterpret_cast<const T*>(P.mptr[P.iB]);
  T* out = reinterpret_cast<T*>(P.out);
  const int shf = P.nH - P.nHF;
  int64_t fkey = -1;
  // B and output bases of tile h (every thread: no barrier)
  auto bases = [&](int64_t hh, int64_t& bb, int64_t& obase) {
    bb = 0;
    obase = 0;
    for (int b = 0; b < P.nH; ++b)
      if ((hh >> b) & 1) {
        bb += P.hs[P.iB][b];
        obase += P.hs[nm][b];
      }
  };
  // B for all s (registers)
  auto loadB = [&](int64_t bb, T (&bv)[RB][NS]) {
    const T* bp = Bm + bb + boff;
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int64_t o = bb + boff + soffB[s] + (r ? P.rbs : 0);
        K4_CHECK(o >= 0 && o < P.span[P.iB], "B element %lld of %lld", (long long)o, (long long)P.span[P.iB]);
        bv[r][s] = __ldg(bp + soffB[s] + (r ? P.rbs : 0));
      }
  };
  int64_t bb, obase;
  T bv[RB][NS];
  bases(h, bb, obase);
  loadB(bb, bv);
  for (; h < h_end; ++h) {
#if K4_PF
    // the next tile's B is in flight while this tile's results are written
    int64_t bbn = 0, obn = 0;
    T bn[RB][NS];
    if (h + 1 < h_end) {
      bases(h + 1, bbn, obn);
      loadB(bbn, bn);
    }
#else
    if (h != blockIdx.x * per) {
      bases(h, bb, obase);
      loadB(bb, bv);
    }
#endif
    if ((h >> shf) != fkey) {
      fkey = h >> shf;
      __syncthreads();   // previous F no longer read
      if (tid < nm) {
        int64_t o = 0;
        for (int b = shf; b < P.nH; ++b)
          if ((h >> b) & 1) o += P.hs[tid][b];
        sbase[tid] = o;
      }
      __syncthreads();
      // F = product of the other members over (F bits, s)
      for (int x = tid; x < nfe; x += NT) {
        T v = {R(1), R(0)};
        const int lo = x & 63, hi = x >> 6;
        for (int j = 0; j < nm; ++j) {
          if (j == P.iB) continue;
          const T* mp = reinterpret_cast<const T*>(P.mptr[j]);
          K4_CHECK(sbase[j] + LUT[j * 128 + lo] + LUT[j * 128 + 64 + hi] < P.span[j], "member %d element %lld", j,
                   (long long)(sbase[j] + LUT[j * 128 + lo] + LUT[j * 128 + 64 + hi]));
          v = cmul(v, __ldg(mp + sbase[j] + LUT[j * 128 + lo] + LUT[j * 128 + 64 + hi]));
        }
        F[x] = v;
      }
      __syncthreads();
    }
    // the results of this tile: 2^NE per thread, the low NEL expansion bits
    // unrolled, the high NEH walked by a rolled loop (NE > 4 only)
    auto emit = [&](int32_t oh, int32_t fh) {
      T* op = out + obase + ob + oh;
#pragma unroll
      for (int e = 0; e < NEVL; ++e) {
        K4_CHECK(fe[e] + fh + NS <= nfe, "F entry %d of %d", fe[e] + fh + NS, nfe);
        const T* fp = F + fe[e] + fh;
        T fr[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) fr[s] = fp[s];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          T acc = cmul(bv[r][0], fr[0]);
#pragma unroll
          for (int s = 1; s < NS; ++s) cfma(acc, bv[r][s], fr[s]);
          const int64_t o = oe[e] + (r ? P.rbo : 0);
          K4_CHECK(obase + ob + oh + o >= 0 && obase + ob + oh + o < P.out_elems, "result %lld of %lld",
                   (long long)(obase + ob + oh + o), (long long)P.out_elems);
          op[o] = acc;
        }
      }
    };
    if constexpr (NEH == 0) {
      emit(0, 0);
    } else {
#pragma unroll 1
      for (int eh = 0; eh < (1 << NEH); ++eh) {
        int32_t oh = 0, fh = 0;
#pragma unroll
        for (int b = 0; b < NEH; ++b)
          if ((eh >> b) & 1) {
            oh += P.oe[NEL + b];
            fh += P.fe[NEL + b] << K;
          }
        emit(oh, fh);
      }
    }
#if K4_PF
    obase = obn;
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int s = 0; s < NS; ++s) bv[r][s] = bn[r][s];
#endif
  }
  if (P.timing && tid == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    atomicMin(&P.timing[2 * P.item], t_start);
    atomicMax(&P.timing[2 * P.item + 1], t_end);
  }
}

template <typename R, int K, int NE, int RB>
const void* fn_k() {
  if constexpr (sizeof(R) == 4)
    return (const void*)k4_kernel_c64<R, K, NE, RB>;
  else
    return (const void*)k4_kernel_c128<R, K, NE, RB>;
}

template <typename R, int K, int RB>
const void* fn_ne(int ne) {
  switch (ne) {
    case 0: return fn_k<R, K, 0, RB>();
    case 1: return fn_k<R, K, 1, RB>();
    case 2: return fn_k<R, K, 2, RB>();
    case 3: return fn_k<R, K, 3, RB>();
    case 4: return fn_k<R, K, 4, RB>();
    case 5: return fn_k<R, K, 5, RB>();
    case 6: return fn_k<R, K, 6, RB>();
    case 7: return fn_k<R, K, 7, RB>();
    default: return fn_k<R, K, 8, RB>();
  }
}

template <typename R>
const void* fn_of(int k, int ne, int rb) {
  if (rb) {
    if (k == 1) return fn_ne<R, 1, 2>(ne);
    if (k == 2) return fn_ne<R, 2, 2>(ne);
    return fn_ne<R, 3, 2>(ne);
  }
  if (k == 1) return fn_ne<R, 1, 1>(ne);
  if (k == 2) return fn_ne<R, 2, 1>(ne);
  return fn_ne<R, 3, 1>(ne);
}

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return qtn_internal_set_error(code, buf);
}

int sm_count() {
  int dev = 0, nsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return nsm;
}

// Plan K4 for `d` (QTN_E_UNSUPPORTED when the item is not an expansion of one
// dominant member); min_e: fewest expansion bits accepted.  nq > 0 (K6): the
// top nq result bits are set aside — not thread, expansion or tile bits; the
// fused kernel walks them per thread (B strides bq, F index bits fq) and the
// plan's output covers the low w - nq bits only.
int make_plan(const qtn_bucket_desc_t* d, int min_e, Plan* P, int* smem, int nq, int ne_max, int ntb) {
  memset(P, 0, sizeof(*P));
  const int w = d->w, k = d->k, nm = d->n_mem;
  const int wf = w - nq;   // free result bits
  const size_t esz = d->dtype == QTN_C64 ? 8 : 16;
  if (d->dtype != QTN_C64 && d->dtype != QTN_C128) return fail(QTN_E_INVALID, "K4: bad dtype");
  if (k < 1 || k > MAXKS || nm < 1 || nm > MAXM || wf < ntb || w > 31 || nq < 0 || nq > MAXQ || ntb < 5 ||
      ntb > TBB)
    return fail(QTN_E_UNSUPPORTED, "K4: w=%d k=%d n_mem=%d nq=%d", w, k, nm, nq);
  // dominant member: most result bits
  int iB = 0, best = -1;
  for (int i = 0; i < nm; ++i) {
    int c = 0;
    for (int b = 0; b < w; ++b) c += d->mem[i].strides[b] != 0;
    if (c > best) best = c, iB = i;
  }
  const qtn_bmember_t& B = d->mem[iB];
  int tb[TBB], nt = 0, eb[MAXE], ne = 0;
  bool carried[64] = {};   // result bits some other member carries
  for (int b = 0; b < w; ++b)
    for (int i = 0; i < nm; ++i)
      if (i != iB && d->mem[i].strides[b] != 0) carried[b] = true;
  int ne_all = 0;   // B-lacking result bits; the lowest ne_max are expansion bits, the rest tile bits
  for (int b = 0; b < wf; ++b)
    if (B.strides[b] == 0) {
      if (ne_all == MAXE) return fail(QTN_E_UNSUPPORTED, "K4: more than %d expansion bits", MAXE);
      ++ne_all;
      if (ne < ne_max) eb[ne++] = b;
    }
  if (wf - ne < ntb) return fail(QTN_E_UNSUPPORTED, "K4: dominant member has %d result bits", best);
  // more than 4 expansion bits (two mid-size members, an outer-product-like
  // expansion): only for wide items — the 45-cone energy's w 22-26 items run
  // 3-5x faster here than in K1, a w = 16 item ran slower (cfg-2: 4 -> 10 us)
  if (ne_all > 4 && w < K4_WIDE_E_MIN_W)
    return fail(QTN_E_UNSUPPORTED, "K4: %d expansion bits at width %d", ne, w);
  // Thread bits.  Lanes (the first 5): B's fastest axes first — one 32-byte
  // sector of B per lane group (2 complex128 / 4 complex64 elements) — then
  // B bits NO other member carries, so every lane of a warp reads the same
  // product-table row (shared-memory broadcast instead of bank conflicts);
  // then the remaining B bits, ascending.  Warps: the next 3.
  bool used[64] = {};
  {
    const int sec = (int)(32 / esz);
    auto take = [&](int b) { tb[nt++] = b; used[b] = true; };
    for (int b = 0; b < wf && nt < ntb; ++b)   // B's local axes 0 .. log2(sec)-1
      if (B.strides[b] != 0 && B.strides[b] < sec) take(b);
    for (int pass = 0; pass < 2; ++pass)
      for (int b = 0; b < wf && nt < 5; ++b)
        if (B.strides[b] != 0 && !used[b] && (pass == 1 || !carried[b])) take(b);
    for (int b = 0; b < wf && nt < ntb; ++b)
      if (B.strides[b] != 0 && !used[b]) take(b);
  }
  if (ne_all < min_e) return fail(QTN_E_UNSUPPORTED, "K4: %d expansion bits", ne_all);
  // replica bit: the first remaining B bit no other member carries (each
  // thread then owns two B coordinates sharing every product-table row —
  // half the shared-memory row reads).  Measured on cfg-2: complex128 all
  // items and complex64 k = 3 gain (w21 k3: 21.3 -> 12.6 us c128, 44 -> 15 us
  // c64); complex64 k <= 2 loses (w24 k2: 46 -> 54 us: 3 blocks/SM instead of 4).
  // Not in fused plans (the set-aside bits already multiply the B registers).
  int rbit = -1;
  if (nq == 0 && (d->dtype == QTN_C128 || k == 3))
    for (int b = 0; b < wf && rbit < 0; ++b)
      if (B.strides[b] != 0 && !used[b] && !carried[b]) rbit = b;
  // tile bits T = tb u eb (u the replica bit); F bits = T bits any other
  // member carries, then the set-aside bits any other member carries
  bool inT[64] = {};
  for (int i = 0; i < nt; ++i) inT[tb[i]] = true;
  for (int i = 0; i < ne; ++i) inT[eb[i]] = true;
  if (rbit >= 0) inT[rbit] = true;
  for (int b = wf; b < w; ++b) inT[b] = true;
  int fbit[64], nf = 0;
  for (int b = 0; b < w; ++b) {
    fbit[b] = -1;
    if (inT[b] && carried[b]) fbit[b] = nf++;
  }
  const int max_fb = d->dtype == QTN_C64 ? MAXFB : MAXFB - 1;
  if (nf + k > max_fb) return fail(QTN_E_UNSUPPORTED, "K4: F table of %d bits", nf + k);
  // member element offsets must fit 32 bits inside a tile's F gathers
  for (int i = 0; i < nm; ++i) {
    if (!d->mem[i].data) return fail(QTN_E_INVALID, "K4: null member %d", i);
    int64_t span = 0;
    for (int b = 0; b < w + k; ++b) span += d->mem[i].strides[b];
    if (span >= ((int64_t)1 << 31)) return fail(QTN_E_UNSUPPORTED, "K4: member %d spans 2^31 elements", i);
    P->mptr[i] = d->mem[i].data;
  }
  if (!d->out && nq == 0) return fail(QTN_E_INVALID, "K4: null output");
  P->out = d->out;
  P->nm = nm;
  P->k = k;
  P->nE = ne;
  P->nF = nf;
  P->iB = iB;
  int nh = 0, nhf = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (int b = 0; b < wf; ++b) {
      if (inT[b]) continue;
      if (carried[b] != (pass == 1)) continue;
      for (int i = 0; i < nm; ++i) P->hs[i][nh] = d->mem[i].strides[b];
      P->hs[nm][nh] = (int64_t)1 << b;
      P->hbit[nh] = (int8_t)b;
      ++nh;
      nhf += carried[b];
    }
  P->nH = nh;
  P->nHF = nhf;
  P->n_tiles = (int64_t)1 << nh;
  P->out_elems = (int64_t)1 << wf;
  for (int i = 0; i < nm; ++i) {
    int64_t sp = 1;
    for (int b = 0; b < w + k; ++b) sp += d->mem[i].strides[b];
    P->span[i] = sp;
  }
  for (int i = 0; i < nm; ++i) {
    if (i == iB) continue;
    for (int q = 0; q < k; ++q) P->fs[i][q] = (uint32_t)d->mem[i].strides[w + q];
    for (int b = 0; b < w; ++b)
      if (fbit[b] >= 0) P->fs[i][k + fbit[b]] = (uint32_t)d->mem[i].strides[b];
  }
  for (int q = 0; q < k; ++q) P->bs[q] = B.strides[w + q];
  for (int i = 0; i < ntb; ++i) {
    P->btb[i] = B.strides[tb[i]];
    P->otb[i] = 1 << tb[i];
    P->ftb[i] = fbit[tb[i]] >= 0 ? 1 << fbit[tb[i]] : 0;
    P->tbit[i] = (int8_t)tb[i];
  }
  for (int i = 0; i < ne; ++i) {
    P->oe[i] = 1 << eb[i];
    P->fe[i] = fbit[eb[i]] >= 0 ? 1 << fbit[eb[i]] : 0;
    P->ebit[i] = (int8_t)eb[i];
  }
  P->nq = nq;
  for (int i = 0; i < nq; ++i) {
    P->bq[i] = B.strides[wf + i];
    P->fq[i] = fbit[wf + i] >= 0 ? 1 << fbit[wf + i] : 0;
  }
  P->rb = rbit >= 0 ? 1 : 0;
  P->rbs = rbit >= 0 ? B.strides[rbit] : 0;
  P->rbo = rbit >= 0 ? (int32_t)1 << rbit : 0;
  *smem = (int)(esz << (nf + k)) + nm * 128 * 4;
  (void)esz;
  return QTN_OK;
}

}  // namespace qtn_k4

size_t qtn_k4_plan_bytes() { return sizeof(qtn_k4::Plan); }

// Program-graph node for one item (qtn_graph_create_host): QTN_E_UNSUPPORTED
// when the item is not a K4 expansion with at least min_e expansion bits.
int qtn_k4_node(const qtn_bucket_desc_t* d, int min_e, unsigned long long* timing, int32_t item, void* plan,
                const void** fn, int* grid, int* smem) {
  using namespace qtn_k4;
  Plan* P = reinterpret_cast<Plan*>(plan);
  int rc = make_plan(d, min_e, P, smem);
  if (rc) return rc;
  P->timing = timing;
  P->item = item;
  *fn = d->dtype == QTN_C64 ? fn_of<float>(P->k, P->nE, P->rb) : fn_of<double>(P->k, P->nE, P->rb);
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, *fn);
  if (e != cudaSuccess) return fail(QTN_E_CUDA, "cudaFuncGetAttributes: %s", cudaGetErrorString(e));
  if (*smem > fa.maxDynamicSharedSizeBytes) {
    e = cudaFuncSetAttribute(*fn, cudaFuncAttributeMaxDynamicSharedMemorySize, *smem);
    if (e != cudaSuccess) return fail(QTN_E_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, *fn, NT, *smem);
  if (e != cudaSuccess) return fail(QTN_E_CUDA, "occupancy: %s", cudaGetErrorString(e));
  if (per_sm < 1) return fail(QTN_E_UNSUPPORTED, "K4 cannot be resident with %d B smem", *smem);
  *grid = (int)std::min<int64_t>(P->n_tiles, (int64_t)per_sm * sm_count());
  return QTN_OK;
}

extern "C" int qtn_bucket_expand(const qtn_bucket_desc_t* d, int32_t min_e, void* stream) {
  using namespace qtn_k4;
  if (!d) return fail(QTN_E_INVALID, "null descriptor");
  static thread_local Plan P;
  const void* fn = nullptr;
  int grid = 0, smem = 0;
  int rc = qtn_k4_node(d, min_e, nullptr, 0, &P, &fn, &grid, &smem);
  if (rc) return rc;
  void* args[] = {&P};
  const cudaError_t e = cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(NT), args, smem, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(QTN_E_CUDA, "K4 launch: %s", cudaGetErrorString(e));
  return QTN_OK;
}

