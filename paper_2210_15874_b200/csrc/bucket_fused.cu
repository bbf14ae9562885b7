// bucket_fused.cu — K6: an expansion item fused with its only consumer.
//
// A consumer item C (one reference bucket, or a merged chain summing k_C <= 3
// indices, src/tensor_core.py:148-164) whose member X is the WHOLE result of
// a producer item P: X carries every result and summed index of C in the
// canonical order, so P's result bits are C's result bits r followed by C's
// summed bits q, and nothing else reads P's result (the reference re-buckets
// it at its earliest index and contracts it there, src/ordering.py:175-187).
//     out_C[r] = sum_q G(q, r) * U(q) * X(q, r)
//     X(q, r)  = sum_s B(s, q, r) * F(f(q, r), s)                 (P, as K4)
// B = P's dominant member, F = the product of P's other members (a per-tile
// table in shared memory, csrc/bucket_expand.cu), U = the product of C's
// members that carry no result index, G = C's one member that does (at most
// one; the widest intermediate of a lightcone is typically read by such a
// pair: cfg-2's w = 24 complex128 result, 268 MB, written and read back by
// two kernels, is never materialised here).
//
// P's K4 plan is made with the q bits set aside: each thread owns one B
// coordinate (8 thread bits), holds B(s, q) for every (s, q) in registers
// (U folded in), and walks its 2^|E| expansion results; per result it forms
// X(q, r) for every q from broadcast product-table rows and sums over q right
// away.  The q loop is ordered so that G is constant over runs of q (the q
// bits G does not carry first): each run is summed, then multiplied by G
// once.  G values are loaded for a whole batch of results before any is
// used.  Sum order: s ascending inside X, q in the plan's order outside; X
// is not rounded to the element type.
//
// One source, three objects (Makefile): K6_PART 0 = planner + C ABI, 1 =
// complex64 kernels, 2 = complex128 kernels (compiled in parallel).
#include "k4_plan.h"

#include <algorithm>
#include <cstdarg>
#include <cstring>

#ifndef K6_PART
#define K6_PART 0
#endif
// L1 prefetch of the next result batch's G lines (cfg-2 w24 pair c128 79.9
// -> 75.8 us, c64 57.4 -> 55.3 us).  Measured and dropped: cp.async staging
// of the next tile's B in shared memory, L2 prefetch of it (neutral).
#ifndef K6_GPF
#define K6_GPF 1
#endif
// expansion bits walked per thread (the producer's other B-lacking bits
// become tile bits: more, smaller tiles balance the persistent grid; 3 and
// 8 measured within 5 % on cfg-2, 2 slower)
#ifndef K6_NE_MAX
#define K6_NE_MAX 8
#endif
// expansion bits unrolled per result batch (at most 2; complex128 with the
// lane split: 1 fits 80 registers, 3 blocks/SM; 2 needs 124, 2 blocks/SM)
#ifndef K6_NEL_C64
#define K6_NEL_C64 2
#endif
#ifndef K6_NEL_C128
#define K6_NEL_C128 2
#endif
// lane-split kernels (two lanes per B coordinate, each with half the q runs)
// for plans with at least two G runs, per element type: bit 0 complex64,
// bit 1 complex128.  cfg-2 w24 pair: complex64 55.3 -> 49.8 us (64 registers,
// 4 blocks/SM); complex128 73.7 -> 69.6 us with one unrolled expansion bit
// (80 registers, 3 blocks/SM; with two it spilled: 77.8 us)
#ifndef K6_SPLIT
#define K6_SPLIT 3
#endif

namespace qtn_k4 {

struct FPlan {
  Plan p;                     // producer plan, q bits set aside; p.out = C's output
  int32_t ng;                 // gathered consumer members (0 or 1)
  const void* gptr;
  int64_t ghs[MAXH];          // G stride of tile bit j (p.hbit order)
  int32_t gtb[TBB];           // of thread bit t
  int32_t ge[MAXE];           // of expansion bit e
  int32_t gq[MAXQ];           // of q loop bit i
  int64_t gspan;
  int32_t nu;                 // consumer members on summed bits only: folded into U[q]
  const void* uptr[MAXM];
  int32_t uq[MAXM][MAXQ];
  int32_t nqn;                // q loop bits G does not carry (the low ones)
  int32_t split;              // lanes per B coordinate (1 or 2)
  int32_t item_c;             // consumer item (timing; p.item = producer)
};

// Kernel selection: K = producer summed bits, NQ = 2^(consumer summed bits),
// GQ = G runs per result (0: no G member), NEL = expansion bits unrolled per
// batch (the rest walked by a rolled loop), SPLIT = lanes per B coordinate.
const void* k6_fn_c64(int k, int nq, int gq, int nel, int split);
const void* k6_fn_c128(int k, int nq, int gq, int nel, int split);

#if K6_PART > 0

__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int m) {
  return {__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m)};
}

// SPLIT = 2: lane bit 4 splits the q runs between the two lanes of a pair
// (each holds half the B file: fewer registers, more resident warps); per
// result batch the pair exchanges half of its per-lane partial results with
// one shuffle step, and each lane stores half of the batch.
template <typename R, int K, int NQ, int GQ, int NEL, int SPLIT>
__device__ __forceinline__ void k6_body(const FPlan& FP) {
  using T = typename Cx<R>::T;
  const Plan& P = FP.p;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int NS = 1 << K;
  constexpr int NR = GQ == 0 ? 1 : GQ;   // runs of q
  constexpr int QN = NQ / NR;            // q per run
  constexpr int NRL = NR / SPLIT;        // runs per lane
  constexpr int NQL = NRL * QN;          // q per lane
  constexpr int NEVL = 1 << NEL;
  static_assert(SPLIT == 1 || (SPLIT == 2 && NR >= 2), "a lane split needs two G runs");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* F = reinterpret_cast<T*>(smem_raw);
  const int nfe = 1 << (P.nF + K);
  uint32_t* LUT = reinterpret_cast<uint32_t*>(smem_raw + sizeof(T) * nfe);
  __shared__ int64_t sbase[MAXM + 1];
  __shared__ T sU[NQ];
  // out / F / G offsets of every batch of the rolled expansion bits
  __shared__ int4 sEH[1 << (MAXE - 1)];
  const int tid = threadIdx.x;
  const int nm = P.nm;
  const int nlo = P.nF + K < 6 ? P.nF + K : 6;
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
  // thread bits (SPLIT 2: lane bit 4 is the run half lr, the others index
  // the plan's 7 thread bits)
  const int lr = SPLIT == 2 ? (tid >> 4) & 1 : 0;
  const int tix = SPLIT == 2 ? ((tid & 15) | ((tid >> 5) << 4)) : tid;
  constexpr int NTB = SPLIT == 2 ? TBB - 1 : TBB;
  int64_t boff = 0;
  int32_t ob = 0, fb = 0, gthr = 0;
#pragma unroll
  for (int b = 0; b < NTB; ++b)
    if ((tix >> b) & 1) {
      boff += P.btb[b];
      ob += P.otb[b];
      fb += P.ftb[b];
      gthr += FP.gtb[b];
    }
  // the low NEL expansion bits: out / F / G offsets per unrolled result
  int32_t oe[NEVL], fe[NEVL], ge[NEVL];
#pragma unroll
  for (int e = 0; e < NEVL; ++e) {
    int32_t o = 0, f = 0, g = 0;
#pragma unroll
    for (int b = 0; b < NEL; ++b)
      if ((e >> b) & 1) {
        o += P.oe[b];
        f += P.fe[b];
        g += FP.ge[b];
      }
    oe[e] = o;
    fe[e] = (fb + f) << K;
    ge[e] = gthr + g;
  }
  // this lane's q values: runs r = rl * SPLIT + lr, q = r * QN + qi
  int64_t qoffB[NQL];
  int32_t fqo[NQL];
#pragma unroll
  for (int ql = 0; ql < NQL; ++ql) {
    const int q = ((ql / QN) * SPLIT + lr) * QN + ql % QN;
    int64_t o = 0;
    int32_t f = 0;
#pragma unroll
    for (int b = 0; b < MAXQ; ++b)
      if ((1 << b) < NQ && ((q >> b) & 1)) {
        o += P.bq[b];
        f += P.fq[b];
      }
    qoffB[ql] = o;
    fqo[ql] = f << K;
  }
  int32_t gro[NRL];   // G offset of each of this lane's runs (a run's q bits are the high loop bits)
#pragma unroll
  for (int rl = 0; rl < NRL; ++rl) {
    const int r = rl * SPLIT + lr;
    int32_t o = 0;
#pragma unroll
    for (int b = 0; b < MAXQ; ++b)
      if ((1 << b) < NQ && (((r * QN) >> b) & 1)) o += FP.gq[b];
    gro[rl] = o;
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
  const int neh = P.nE - NEL;   // expansion bits walked by the rolled loop
  for (int eh = tid; eh < (1 << neh); eh += NT) {
    int32_t oh = 0, fh = 0, gh = 0;
    for (int b = 0; b < neh; ++b)
      if ((eh >> b) & 1) {
        oh += P.oe[NEL + b];
        fh += P.fe[NEL + b] << K;
        gh += FP.ge[NEL + b];
      }
    sEH[eh] = make_int4(oh, fh, gh, 0);
  }
  // balanced contiguous runs of tile ids (every block gets floor or ceil)
  int64_t h = (int64_t)blockIdx.x * P.n_tiles / gridDim.x;
  const int64_t h_end = ((int64_t)blockIdx.x + 1) * P.n_tiles / gridDim.x;
  if (h >= h_end) return;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  unsigned long long t_start = 0;
  if (P.timing && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  // U[q] = product of the consumer members that carry no result bit
  if (tid < NQ) {
    T u = {R(1), R(0)};
    for (int i = 0; i < FP.nu; ++i) {
      int32_t o = 0;
#pragma unroll
      for (int b = 0; b < MAXQ; ++b)
        if ((tid >> b) & 1) o += FP.uq[i][b];
      u = cmul(u, __ldg(reinterpret_cast<const T*>(FP.uptr[i]) + o));
    }
    sU[tid] = u;
  }
  __syncthreads();
  const T* Bm = reinterpret_cast<const T*>(P.mptr[P.iB]);
  const T* Gm = reinterpret_cast<const T*>(FP.gptr);
  T* out = reinterpret_cast<T*>(P.out);
  const int shf = P.nH - P.nHF;
  int64_t fkey = -1;
  for (; h < h_end; ++h) {
    int64_t bb = 0, obase = 0, gb = 0;
    for (int b = 0; b < P.nH; ++b)
      if ((h >> b) & 1) {
        bb += P.hs[P.iB][b];
        obase += P.hs[nm][b];
        gb += FP.ghs[b];
      }
    // B for every (q, s) of this lane: NQL * NS independent loads in flight, U folded in
    T bv[NQL][NS];
    {
      const T* bp = Bm + bb + boff;
#pragma unroll
      for (int ql = 0; ql < NQL; ++ql)
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          K4_CHECK(bb + boff + qoffB[ql] + soffB[s] >= 0 && bb + boff + qoffB[ql] + soffB[s] < P.span[P.iB],
                   "K6 B element %lld", (long long)(bb + boff + qoffB[ql] + soffB[s]));
          bv[ql][s] = __ldg(bp + qoffB[ql] + soffB[s]);
        }
      if (FP.nu) {
#pragma unroll
        for (int ql = 0; ql < NQL; ++ql) {
          const T u = sU[((ql / QN) * SPLIT + lr) * QN + ql % QN];
#pragma unroll
          for (int s = 0; s < NS; ++s) bv[ql][s] = cmul(u, bv[ql][s]);
        }
      }
    }
    if ((h >> shf) != fkey) {
      fkey = h >> shf;
      __syncthreads();
      if (tid < nm) {
        int64_t o = 0;
        for (int b = shf; b < P.nH; ++b)
          if ((h >> b) & 1) o += P.hs[tid][b];
        sbase[tid] = o;
      }
      __syncthreads();
      for (int x = tid; x < nfe; x += NT) {
        T v = {R(1), R(0)};
        const int lo = x & 63, hi = x >> 6;
        for (int j = 0; j < nm; ++j) {
          if (j == P.iB) continue;
          const T* mp = reinterpret_cast<const T*>(P.mptr[j]);
          K4_CHECK(sbase[j] + LUT[j * 128 + lo] + LUT[j * 128 + 64 + hi] < P.span[j], "K6 member %d", j);
          v = cmul(v, __ldg(mp + sbase[j] + LUT[j * 128 + lo] + LUT[j * 128 + 64 + hi]));
        }
        F[x] = v;
      }
      __syncthreads();
    }
    T* op = out + obase + ob;
    const T* gp = Gm + gb;
    // batches of NEVL results: the high expansion bits walked here
#pragma unroll 1
    for (int eh = 0; eh < (1 << neh); ++eh) {
      const int4 ehv = sEH[eh];
      const int32_t oh = ehv.x, fh = ehv.y, gh = ehv.z;
      // G for the whole batch first (one long-latency round trip per batch);
      // the next batch's lines are prefetched into L1 meanwhile
      T gv[NEVL][NRL];
#if K6_GPF
      if constexpr (GQ > 0) {
        if (eh + 1 < (1 << neh)) {
          const int32_t ghn = sEH[eh + 1].z;
#pragma unroll
          for (int e = 0; e < NEVL; ++e)
#pragma unroll
            for (int rl = 0; rl < NRL; ++rl) prefetch_l1(gp + ge[e] + ghn + gro[rl]);
        }
      }
#endif
      if constexpr (GQ > 0) {
#pragma unroll
        for (int e = 0; e < NEVL; ++e)
#pragma unroll
          for (int rl = 0; rl < NRL; ++rl) {
            K4_CHECK(gb + ge[e] + gh + gro[rl] >= 0 && gb + ge[e] + gh + gro[rl] < FP.gspan, "K6 G element %lld",
                     (long long)(gb + ge[e] + gh + gro[rl]));
            gv[e][rl] = __ldg(gp + ge[e] + gh + gro[rl]);
          }
      }
      // per result: this lane's runs, G applied per run
      T acc[NEVL];
#pragma unroll
      for (int e = 0; e < NEVL; ++e) {
        const T* fpe = F + fe[e] + fh;
#pragma unroll
        for (int rl = 0; rl < NRL; ++rl) {
          T xs;
#pragma unroll
          for (int qi = 0; qi < QN; ++qi) {
            const int ql = rl * QN + qi;
            const T* fp = fpe + fqo[ql];
            K4_CHECK(fe[e] + fh + fqo[ql] + NS <= nfe, "K6 F entry %d of %d", fe[e] + fh + fqo[ql] + NS, nfe);
            if (qi == 0)
              xs = cmul(bv[ql][0], fp[0]);
            else
              cfma(xs, bv[ql][0], fp[0]);
#pragma unroll
            for (int s = 1; s < NS; ++s) cfma(xs, bv[ql][s], fp[s]);
          }
          if constexpr (GQ > 0) {
            if (rl == 0)
              acc[e] = cmul(gv[e][rl], xs);
            else
              cfma(acc[e], gv[e][rl], xs);
          } else {
            acc[e] = xs;
          }
        }
      }
      if constexpr (SPLIT == 1) {
#pragma unroll
        for (int e = 0; e < NEVL; ++e) {
          K4_CHECK(obase + ob + oh + oe[e] >= 0 && obase + ob + oh + oe[e] < P.out_elems, "K6 result %lld",
                   (long long)(obase + ob + oh + oe[e]));
          op[oh + oe[e]] = acc[e];
        }
      } else if constexpr (NEVL == 1) {
        // both lanes hold the same result: the run-0 lane adds its partner's
        const T o = shfl_xor(acc[0], 16);
        if (lr == 0) op[oh + oe[0]] = T{acc[0].x + o.x, acc[0].y + o.y};
      } else {
        // reduce-scatter over the lane pair: lane lr keeps results
        // [lr * HALF, lr * HALF + HALF), run-0 partial first
        constexpr int HALF = NEVL / 2;
#pragma unroll
        for (int j = 0; j < HALF; ++j) {
          const T keep = lr ? acc[HALF + j] : acc[j];
          const T send = lr ? acc[j] : acc[HALF + j];
          const T o = shfl_xor(send, 16);
          const T v = lr ? T{o.x + keep.x, o.y + keep.y} : T{keep.x + o.x, keep.y + o.y};
          const int32_t oo = lr ? oe[HALF + j] : oe[j];
          K4_CHECK(obase + ob + oh + oo >= 0 && obase + ob + oh + oo < P.out_elems, "K6 result %lld",
                   (long long)(obase + ob + oh + oo));
          op[oh + oo] = v;
        }
      }
    }
  }
  if (P.timing && tid == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    atomicMin(&P.timing[2 * P.item], t_start);
    atomicMax(&P.timing[2 * P.item + 1], t_end);
    atomicMin(&P.timing[2 * FP.item_c], t_start);
    atomicMax(&P.timing[2 * FP.item_c + 1], t_end);
  }
}

#ifndef K6_MINB_C64
#define K6_MINB_C64 3
#endif
#ifndef K6_MINB_C128
#define K6_MINB_C128 2
#endif
#ifndef K6_MINB_SPLIT_C64
#define K6_MINB_SPLIT_C64 4
#endif
// complex128 split kernels: 2 blocks/SM with two unrolled expansion bits (124
// registers, more loads in flight per thread) measured 1 % faster on cfg-2
// than 3 blocks/SM with one (80 registers)
#ifndef K6_MINB_SPLIT_C128
#define K6_MINB_SPLIT_C128 2
#endif
#if K6_PART == 1
using KR = float;
#define K6_MINB K6_MINB_C64
#define K6_MINB_SPLIT K6_MINB_SPLIT_C64
#define K6_KERNEL k6_kernel_c64
#define K6_FN k6_fn_c64
#else
using KR = double;
#define K6_MINB K6_MINB_C128
#define K6_MINB_SPLIT K6_MINB_SPLIT_C128
#define K6_KERNEL k6_kernel_c128
#define K6_FN k6_fn_c128
#endif

template <int K, int NQ, int GQ, int NEL, int SPLIT>
__global__ void __launch_bounds__(NT, SPLIT == 2 ? K6_MINB_SPLIT : K6_MINB) K6_KERNEL(const __grid_constant__ FPlan FP) {
  k6_body<KR, K, NQ, GQ, NEL, SPLIT>(FP);
}

// kernel selectors: internal linkage — part 1 and part 2 instantiate the same
// helper names for different kernels, and the linker must not merge them
namespace {

template <int K, int NQ, int GQ, int SPLIT>
const void* fn_nel(int nel) {
  if (nel == 0) return (const void*)K6_KERNEL<K, NQ, GQ, 0, SPLIT>;
  if (nel == 1) return (const void*)K6_KERNEL<K, NQ, GQ, 1, SPLIT>;
  return (const void*)K6_KERNEL<K, NQ, GQ, 2, SPLIT>;
}

template <int K, int NQ, int GQ>
const void* fn_split(int nel, int split) {
  if constexpr (GQ >= 2) {
    if (split == 2) return fn_nel<K, NQ, GQ, 2>(nel);
  }
  return split == 1 ? fn_nel<K, NQ, GQ, 1>(nel) : nullptr;
}

template <int K, int NQ>
const void* fn_gq(int gq, int nel, int split) {
  if (gq == 0) return fn_split<K, NQ, 0>(nel, split);
  if (gq == 1) return fn_split<K, NQ, 1>(nel, split);
  if (gq == 2 && NQ >= 2) return fn_split<K, NQ, (NQ >= 2 ? 2 : 1)>(nel, split);
  if (gq == 4 && NQ >= 4) return fn_split<K, NQ, (NQ >= 4 ? 4 : 1)>(nel, split);
  if (gq == 8 && NQ >= 8) return fn_split<K, NQ, (NQ >= 8 ? 8 : 1)>(nel, split);
  return nullptr;
}

}  // namespace

// B file: NQ * 2^K values per thread, at most 16
const void* K6_FN(int k, int nq, int gq, int nel, int split) {
  if (k == 1 && nq == 2) return fn_gq<1, 2>(gq, nel, split);
  if (k == 1 && nq == 4) return fn_gq<1, 4>(gq, nel, split);
  if (k == 1 && nq == 8) return fn_gq<1, 8>(gq, nel, split);
  if (k == 2 && nq == 2) return fn_gq<2, 2>(gq, nel, split);
  if (k == 2 && nq == 4) return fn_gq<2, 4>(gq, nel, split);
  if (k == 3 && nq == 2) return fn_gq<3, 2>(gq, nel, split);
  return nullptr;
}

#endif  // K6_PART > 0

#if K6_PART == 0

// Plan K6 for producer `dp` feeding member `ipc` of consumer `dc`.
// QTN_E_UNSUPPORTED when the pair does not have that shape or the producer is
// not a K4 expansion once the consumer's summed bits are set aside.
int make_fplan(const qtn_bucket_desc_t* dp, const qtn_bucket_desc_t* dc, int ipc, FPlan* F, int* smem) {
  memset(F, 0, sizeof(*F));
  if (!dp || !dc) return fail(QTN_E_INVALID, "K6: null descriptor");
  const int wc = dc->w, kc = dc->k, nmc = dc->n_mem;
  if (dc->dtype != dp->dtype) return fail(QTN_E_INVALID, "K6: producer and consumer dtypes differ");
  if (kc < 1 || kc > MAXQ || nmc < 1 || nmc > MAXM || ipc < 0 || ipc >= nmc || dp->w != wc + kc)
    return fail(QTN_E_UNSUPPORTED, "K6: consumer w=%d k=%d n_mem=%d, producer w=%d", wc, kc, nmc, dp->w);
  // the producer's result is the consumer's member ipc in canonical order
  if (dc->mem[ipc].data != dp->out) return fail(QTN_E_INVALID, "K6: consumer member %d is not the producer's result", ipc);
  for (int b = 0; b < wc + kc; ++b)
    if (dc->mem[ipc].strides[b] != ((int64_t)1 << b))
      return fail(QTN_E_UNSUPPORTED, "K6: consumer member %d is not the whole producer result", ipc);
  if ((1 << kc) * (1 << dp->k) > 16)
    return fail(QTN_E_UNSUPPORTED, "K6: %d B registers per thread", (1 << kc) * (1 << dp->k));
  // lane split (K6_SPLIT, per element type) when G runs exist — decided from
  // the consumer members before the producer plan (7 thread bits)
  int ng = 0;
  bool gcarries_q = false;
  for (int i = 0; i < nmc; ++i) {
    if (i == ipc) continue;
    bool res = false;
    for (int b = 0; b < wc; ++b) res |= dc->mem[i].strides[b] != 0;
    if (res) {
      ++ng;
      for (int q = 0; q < kc; ++q) gcarries_q |= dc->mem[i].strides[wc + q] != 0;
    }
  }
  const int split = (ng == 1 && gcarries_q && ((K6_SPLIT >> (dp->dtype == QTN_C128 ? 1 : 0)) & 1)) ? 2 : 1;
  int rc = make_plan(dp, 0, &F->p, smem, kc, K6_NE_MAX, split == 2 ? TBB - 1 : TBB);
  if (rc) return rc;
  F->split = split;
  Plan& P = F->p;
  if (!dc->out) return fail(QTN_E_INVALID, "K6: null output");
  P.out = dc->out;
  for (int i = 0; i < nmc; ++i) {
    if (i == ipc) continue;
    const qtn_bmember_t& m = dc->mem[i];
    if (!m.data) return fail(QTN_E_INVALID, "K6: null consumer member %d", i);
    bool res = false;
    int64_t span = 1;
    for (int b = 0; b < wc + kc; ++b) span += m.strides[b];
    for (int b = 0; b < wc; ++b) res |= m.strides[b] != 0;
    if (span >= ((int64_t)1 << 31)) return fail(QTN_E_UNSUPPORTED, "K6: consumer member %d spans 2^31 elements", i);
    if (res) {
      if (F->ng) return fail(QTN_E_UNSUPPORTED, "K6: more than one consumer member carries result bits");
      F->ng = 1;
      F->gptr = m.data;
      for (int j = 0; j < P.nH; ++j) F->ghs[j] = m.strides[P.hbit[j]];
      for (int t = 0; t < TBB; ++t) F->gtb[t] = (int32_t)m.strides[P.tbit[t]];
      for (int e = 0; e < P.nE; ++e) F->ge[e] = (int32_t)m.strides[P.ebit[e]];
      for (int q = 0; q < kc; ++q) F->gq[q] = (int32_t)m.strides[wc + q];
      F->gspan = span;
    } else {
      const int u = F->nu++;
      F->uptr[u] = m.data;
      for (int q = 0; q < kc; ++q) F->uq[u][q] = (int32_t)m.strides[wc + q];
    }
  }
  // q loop order: the bits G does not carry first (G is then constant over
  // runs of 2^nqn consecutive q)
  int ord[MAXQ], no = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (int q = 0; q < kc; ++q) {
      const bool carried = F->ng && F->gq[q] != 0;
      if (carried == (pass == 1)) ord[no++] = q;
      if (!carried && pass == 0) ++F->nqn;
    }
  {
    const FPlan T0 = *F;
    for (int i = 0; i < kc; ++i) {
      P.bq[i] = T0.p.bq[ord[i]];
      P.fq[i] = T0.p.fq[ord[i]];
      F->gq[i] = T0.gq[ord[i]];
      for (int u = 0; u < F->nu; ++u) F->uq[u][i] = T0.uq[u][ord[i]];
    }
  }
  return QTN_OK;
}

// the kernel of a plan (nullptr: no instantiation)
const void* fn_of_plan(const FPlan& F, int dtype) {
  const int nq = 1 << F.p.nq;
  const int gq = F.ng ? (nq >> F.nqn) : 0;
  const int nel_max = dtype == QTN_C64 ? K6_NEL_C64 : K6_NEL_C128;
  const int nel = F.p.nE < nel_max ? F.p.nE : nel_max;
  return dtype == QTN_C64 ? k6_fn_c64(F.p.k, nq, gq, nel, F.split) : k6_fn_c128(F.p.k, nq, gq, nel, F.split);
}

}  // namespace qtn_k4

size_t qtn_k6_plan_bytes() { return sizeof(qtn_k4::FPlan); }

// Program-graph node for a producer / consumer pair (qtn_graph_create_host).
int qtn_k6_node(const qtn_bucket_desc_t* dp, const qtn_bucket_desc_t* dc, int ipc, unsigned long long* timing,
                int32_t item_p, int32_t item_c, void* plan, const void** fn, int* grid, int* smem) {
  using namespace qtn_k4;
  FPlan* F = reinterpret_cast<FPlan*>(plan);
  int rc = make_fplan(dp, dc, ipc, F, smem);
  if (rc) return rc;
  F->p.timing = timing;
  F->p.item = item_p;
  F->item_c = item_c;
  *fn = fn_of_plan(*F, dp->dtype);
  if (!*fn) return fail(QTN_E_UNSUPPORTED, "K6: no kernel for k=%d nq=%d", F->p.k, F->p.nq);
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
  if (per_sm < 1) return fail(QTN_E_UNSUPPORTED, "K6 cannot be resident with %d B smem", *smem);
  *grid = (int)std::min<int64_t>(F->p.n_tiles, (int64_t)per_sm * sm_count());
  return QTN_OK;
}

extern "C" int qtn_bucket_expand_fused_plan(const qtn_bucket_desc_t* producer, const qtn_bucket_desc_t* consumer,
                                            int32_t member, int32_t* info) {
  using namespace qtn_k4;
  if (!info) return fail(QTN_E_INVALID, "null info");
  static thread_local FPlan F;
  int smem = 0;
  const int rc = make_fplan(producer, consumer, member, &F, &smem);
  if (rc) return rc;
  if (!fn_of_plan(F, producer->dtype)) return fail(QTN_E_UNSUPPORTED, "K6: no kernel for k=%d nq=%d", F.p.k, F.p.nq);
  info[0] = F.p.k;
  info[1] = F.p.nq;
  info[2] = F.p.nE;
  info[3] = F.p.nF;
  info[4] = F.ng;
  info[5] = F.nu;
  info[6] = F.nqn;
  info[7] = F.p.nH;
  return QTN_OK;
}

extern "C" int qtn_bucket_expand_fused(const qtn_bucket_desc_t* producer, const qtn_bucket_desc_t* consumer,
                                       int32_t member, void* stream) {
  using namespace qtn_k4;
  static thread_local FPlan F;
  const void* fn = nullptr;
  int grid = 0, smem = 0;
  int rc = qtn_k6_node(producer, consumer, member, nullptr, 0, 0, &F, &fn, &grid, &smem);
  if (rc) return rc;
  void* args[] = {&F};
  const cudaError_t e = cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(NT), args, smem, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(QTN_E_CUDA, "K6 launch: %s", cudaGetErrorString(e));
  return QTN_OK;
}

#else

}  // namespace qtn_k4

#endif  // K6_PART == 0
