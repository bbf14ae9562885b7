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

int qtn_internal_set_error(int code, const char* msg);

// QTN_DEBUG build: bounds-check every member / product-table / result index
#ifdef QTN_DEBUG
#define K4_CHECK(cond, ...)                                                        \
  do {                                                                             \
    if (!(cond)) {                                                                 \
      printf("K4_CHECK %s:%d (block %d thread %d): ", __FILE__, __LINE__,          \
             (int)blockIdx.x, (int)threadIdx.x);                                   \
      printf(__VA_ARGS__);                                                         \
      printf("\n");                                                               \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define K4_CHECK(cond, ...) \
  do {                      \
  } while (0)
#endif

namespace qtn_k4 {

constexpr int NT = 256;
constexpr int TBB = 8;                  // thread bits (log2 NT)
constexpr int MAXE = 8;                 // expansion bits (the low 4 unrolled per thread, the rest rolled)
constexpr int K4_WIDE_E_MIN_W = 20;     // more than 4 expansion bits: widths from here
constexpr int MAXKS = 3;                // summed bits
constexpr int MAXFB = 12;               // F table bits (|F| + k)
constexpr int MAXM = QTN_MAX_MEMBERS;
constexpr int MAXH = 32;                // tile-selecting result bits
constexpr int MAXQ = 3;                 // K6: consumer summed bits (set-aside producer bits)

struct Plan {
  void* out;
  const void* mptr[MAXM];
  int32_t nm, k, nE, nF, nH, iB;
  int32_t nHF;                          // tile-id bits other members carry (the highest nHF of nH)
  int64_t n_tiles;
  int64_t out_elems;                    // 2^w
  int64_t span[MAXM];                   // elements each member spans (QTN_DEBUG bounds checks)
  int64_t hs[MAXM + 1][MAXH];           // per member (and out, index nm): stride of tile bit j
  uint32_t fs[MAXM][MAXFB];             // F entry bit q (s bits first) -> member stride
  int64_t bs[MAXKS];                    // B strides of the summed bits
  int64_t btb[TBB];                     // B strides of the thread bits
  int32_t otb[TBB], ftb[TBB];           // out stride / F index bit of the thread bits
  int32_t oe[MAXE], fe[MAXE];           // out stride / F index bit of the expansion bits
  int32_t rb;                           // replica bit present (RB = 2): a B bit no other member carries
  int64_t rbs;                          // its B stride
  int32_t rbo;                          // its output stride
  unsigned long long* timing;
  int32_t item;
  // result bit of every thread / expansion / tile bit (fused plans map a
  // consumer's members onto the same bits); the nq set-aside bits (K6)
  int8_t tbit[TBB], ebit[MAXE], hbit[MAXH];
  int32_t nq;                           // top result bits set aside (K6: the consumer's summed bits)
  int64_t bq[MAXQ];                     // B stride of set-aside bit i
  int32_t fq[MAXQ];                     // F index bit (1 << f) of set-aside bit i, 0 = no other member carries it
};

template <typename R> struct Cx;
template <> struct Cx<float> { using T = float2; };
template <> struct Cx<double> { using T = double2; };

template <typename T>
__device__ __forceinline__ T cmul(T a, T b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T>
__device__ __forceinline__ void cfma(T& acc, T a, T b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}

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

// =========================================================================
// K6: an expansion item fused with its only consumer
// =========================================================================
// A consumer item C whose member X is the whole result of a K4-shaped
// producer item P (X carries every result and summed bit of C, so P's result
// bits are C's result bits r followed by C's summed bits q):
//     out_C[r] = sum_q G(q, r) * X(q, r),   X(q, r) = sum_s B(s, q, r) * F(f(q, r), s)
// G = the product of C's other members.  P's K4 plan is made with the q bits
// set aside: each thread loads B for every (q, s) into registers, forms X(q,
// r) for its results in registers and sums over q right away — X (the widest
// intermediate of a lightcone: 2^24 complex128 = 268 MB at cfg-2) is never
// written to or read back from HBM.  Products and sums follow the unfused
// order (s ascending inside X, q ascending outside); X is not rounded to the
// element type in between.
constexpr int MAXG = 2;   // consumer members carrying result bits (gathered per result)

struct FPlan {
  Plan p;                     // producer plan, q bits set aside; p.out = C's output
  int32_t ng;                 // gathered consumer members
  const void* gptr[MAXG];
  int64_t ghs[MAXG][MAXH];    // stride of tile bit j (p.hbit order)
  int32_t gtb[MAXG][TBB];     // stride of thread bit t
  int32_t ge[MAXG][MAXE];     // stride of expansion bit e
  int32_t gq[MAXG][MAXQ];     // stride of consumer summed bit i
  int64_t gspan[MAXG];
  int32_t nu;                 // consumer members on summed bits only: folded into U[q]
  const void* uptr[MAXM];
  int32_t uq[MAXM][MAXQ];
  int32_t item_c;             // consumer item (timing; p.item = producer)
};

template <typename R, int K, int NE, int NQ>
__device__ __forceinline__ void k6_body(const FPlan& FP);

template <typename R, int K, int NE, int NQ>
__global__ void __launch_bounds__(NT, 2) k6_kernel_c64(const __grid_constant__ FPlan FP) {
  k6_body<R, K, NE, NQ>(FP);
}
template <typename R, int K, int NE, int NQ>
__global__ void __launch_bounds__(NT, 2) k6_kernel_c128(const __grid_constant__ FPlan FP) {
  k6_body<R, K, NE, NQ>(FP);
}

template <typename R, int K, int NE, int NQ>
__device__ __forceinline__ void k6_body(const FPlan& FP) {
  using T = typename Cx<R>::T;
  const Plan& P = FP.p;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int NS = 1 << K;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* F = reinterpret_cast<T*>(smem_raw);
  const int nfe = 1 << (P.nF + K);
  uint32_t* LUT = reinterpret_cast<uint32_t*>(smem_raw + sizeof(T) * nfe);
  __shared__ int64_t sbase[MAXM + 1];
  __shared__ T sU[NQ];
  const int tid = threadIdx.x;
  const int nm = P.nm;
  const int ng = FP.ng;
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
  int64_t boff = 0;
  int32_t ob = 0, fb = 0;
  int32_t gthr[MAXG] = {};
#pragma unroll
  for (int b = 0; b < TBB; ++b)
    if ((tid >> b) & 1) {
      boff += P.btb[b];
      ob += P.otb[b];
      fb += P.ftb[b];
#pragma unroll
      for (int g = 0; g < MAXG; ++g) gthr[g] += FP.gtb[g][b];
    }
  // the low 2 expansion bits unrolled (the B file already holds NQ * NS
  // values), the rest walked by a rolled loop
  constexpr int NEL = NE < 2 ? NE : 2;
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
  int64_t soffB[NS], qoffB[NQ];
  int32_t fqo[NQ];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    int64_t o = 0;
#pragma unroll
    for (int b = 0; b < K; ++b)
      if ((s >> b) & 1) o += P.bs[b];
    soffB[s] = o;
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    int64_t o = 0;
    int32_t f = 0;
#pragma unroll
    for (int b = 0; b < MAXQ; ++b)
      if ((1 << b) < NQ && ((q >> b) & 1)) {
        o += P.bq[b];
        f += P.fq[b];
      }
    qoffB[q] = o;
    fqo[q] = f << K;
  }
  const int64_t per = (P.n_tiles + gridDim.x - 1) / gridDim.x;
  int64_t h = (int64_t)blockIdx.x * per;
  const int64_t h_end = h + per < P.n_tiles ? h + per : P.n_tiles;
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
  T* out = reinterpret_cast<T*>(P.out);
  const int shf = P.nH - P.nHF;
  int64_t fkey = -1;
  for (; h < h_end; ++h) {
    int64_t bb = 0, obase = 0;
    int64_t gb[MAXG] = {};
    for (int b = 0; b < P.nH; ++b)
      if ((h >> b) & 1) {
        bb += P.hs[P.iB][b];
        obase += P.hs[nm][b];
#pragma unroll
        for (int g = 0; g < MAXG; ++g) gb[g] += FP.ghs[g][b];
      }
    // B for every (q, s): NQ * NS independent loads in flight
    T bv[NQ][NS];
    {
      const T* bp = Bm + bb + boff;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          K4_CHECK(bb + boff + qoffB[q] + soffB[s] >= 0 && bb + boff + qoffB[q] + soffB[s] < P.span[P.iB],
                   "K6 B element %lld", (long long)(bb + boff + qoffB[q] + soffB[s]));
          bv[q][s] = __ldg(bp + qoffB[q] + soffB[s]);
        }
      // U[q] folded into the B file (NQ * NS products per tile instead of
      // one per result and q)
      if (FP.nu) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const T u = sU[q];
#pragma unroll
          for (int s = 0; s < NS; ++s) bv[q][s] = cmul(u, bv[q][s]);
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
    auto emit = [&](int32_t oh, int32_t fh, const int32_t (&gh)[MAXG]) {
      T* op = out + obase + ob + oh;
#pragma unroll
      for (int e = 0; e < NEVL; ++e) {
        int32_t ge[MAXG];
#pragma unroll
        for (int g = 0; g < MAXG; ++g) {
          int32_t o = gthr[g] + gh[g];
#pragma unroll
          for (int b = 0; b < NEL; ++b)
            if ((e >> b) & 1) o += FP.ge[g][b];
          ge[g] = o;
        }
        T acc;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const T* fp = F + fe[e] + fh + fqo[q];
          K4_CHECK(fe[e] + fh + fqo[q] + NS <= nfe, "K6 F entry %d of %d", fe[e] + fh + fqo[q] + NS, nfe);
          T x = cmul(bv[q][0], fp[0]);
#pragma unroll
          for (int s = 1; s < NS; ++s) cfma(x, bv[q][s], fp[s]);
#pragma unroll
          for (int gi = 0; gi < MAXG; ++gi)
            if (gi < ng) {
              int32_t o = ge[gi];
#pragma unroll
              for (int b = 0; b < MAXQ; ++b)
                if ((1 << b) < NQ && ((q >> b) & 1)) o += FP.gq[gi][b];
              K4_CHECK(gb[gi] + o >= 0 && gb[gi] + o < FP.gspan[gi], "K6 consumer member %d element %lld", gi,
                       (long long)(gb[gi] + o));
              x = cmul(__ldg(reinterpret_cast<const T*>(FP.gptr[gi]) + gb[gi] + o), x);
            }
          if (q == 0) {
            acc = x;
          } else {
            acc.x += x.x;
            acc.y += x.y;
          }
        }
        K4_CHECK(obase + ob + oh + oe[e] >= 0 && obase + ob + oh + oe[e] < P.out_elems, "K6 result %lld",
                 (long long)(obase + ob + oh + oe[e]));
        op[oe[e]] = acc;
      }
    };
    if constexpr (NEH == 0) {
      const int32_t gh[MAXG] = {};
      emit(0, 0, gh);
    } else {
#pragma unroll 1
      for (int eh = 0; eh < (1 << NEH); ++eh) {
        int32_t oh = 0, fh = 0;
        int32_t gh[MAXG] = {};
#pragma unroll
        for (int b = 0; b < NEH; ++b)
          if ((eh >> b) & 1) {
            oh += P.oe[NEL + b];
            fh += P.fe[NEL + b] << K;
#pragma unroll
            for (int g = 0; g < MAXG; ++g) gh[g] += FP.ge[g][NEL + b];
          }
        emit(oh, fh, gh);
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

// register budget of the B file: NQ * 2^K values per thread
template <typename R, int K, int NQ>
constexpr bool k6_fits() {
  return NQ * (1 << K) <= (sizeof(R) == 4 ? 32 : 16);
}

template <typename R, int K, int NE, int NQ>
const void* fn_k6e() {
  if constexpr (!k6_fits<R, K, NQ>())
    return nullptr;
  else if constexpr (sizeof(R) == 4)
    return (const void*)k6_kernel_c64<R, K, NE, NQ>;
  else
    return (const void*)k6_kernel_c128<R, K, NE, NQ>;
}

template <typename R, int K, int NQ>
const void* fn_k6_ne(int ne) {
  switch (ne) {
    case 0: return fn_k6e<R, K, 0, NQ>();
    case 1: return fn_k6e<R, K, 1, NQ>();
    case 2: return fn_k6e<R, K, 2, NQ>();
    case 3: return fn_k6e<R, K, 3, NQ>();
    case 4: return fn_k6e<R, K, 4, NQ>();
    case 5: return fn_k6e<R, K, 5, NQ>();
    case 6: return fn_k6e<R, K, 6, NQ>();
    case 7: return fn_k6e<R, K, 7, NQ>();
    default: return fn_k6e<R, K, 8, NQ>();
  }
}

template <typename R, int K>
const void* fn_k6_q(int nq, int ne) {
  if (nq == 1) return fn_k6_ne<R, K, 2>(ne);
  if (nq == 2) return fn_k6_ne<R, K, 4>(ne);
  return fn_k6_ne<R, K, 8>(ne);
}

template <typename R>
const void* fn_k6(int k, int nq, int ne) {
  if (k == 1) return fn_k6_q<R, 1>(nq, ne);
  if (k == 2) return fn_k6_q<R, 2>(nq, ne);
  return fn_k6_q<R, 3>(nq, ne);
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
int make_plan(const qtn_bucket_desc_t* d, int min_e, Plan* P, int* smem, int nq = 0) {
  memset(P, 0, sizeof(*P));
  const int w = d->w, k = d->k, nm = d->n_mem;
  const int wf = w - nq;   // free result bits
  const size_t esz = d->dtype == QTN_C64 ? 8 : 16;
  if (d->dtype != QTN_C64 && d->dtype != QTN_C128) return fail(QTN_E_INVALID, "K4: bad dtype");
  if (k < 1 || k > MAXKS || nm < 1 || nm > MAXM || wf < TBB || w > 31 || nq < 0 || nq > MAXQ)
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
  for (int b = 0; b < wf; ++b)
    if (B.strides[b] == 0) {
      if (ne == MAXE) return fail(QTN_E_UNSUPPORTED, "K4: more than %d expansion bits", MAXE);
      eb[ne++] = b;
    }
  if (wf - ne < TBB) return fail(QTN_E_UNSUPPORTED, "K4: dominant member has %d result bits", best);
  // more than 4 expansion bits (two mid-size members, an outer-product-like
  // expansion): only for wide items — the 45-cone energy's w 22-26 items run
  // 3-5x faster here than in K1, a w = 16 item ran slower (cfg-2: 4 -> 10 us)
  if (ne > 4 && w < K4_WIDE_E_MIN_W)
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
    for (int b = 0; b < wf && nt < TBB; ++b)   // B's local axes 0 .. log2(sec)-1
      if (B.strides[b] != 0 && B.strides[b] < sec) take(b);
    for (int pass = 0; pass < 2; ++pass)
      for (int b = 0; b < wf && nt < 5; ++b)
        if (B.strides[b] != 0 && !used[b] && (pass == 1 || !carried[b])) take(b);
    for (int b = 0; b < wf && nt < TBB; ++b)
      if (B.strides[b] != 0 && !used[b]) take(b);
  }
  if (ne < min_e) return fail(QTN_E_UNSUPPORTED, "K4: %d expansion bits", ne);
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
  for (int i = 0; i < TBB; ++i) {
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

// Plan K6 for producer `dp` feeding member `ipc` of consumer `dc` (see
// k6_body).  QTN_E_UNSUPPORTED when the pair does not have that shape or the
// producer is not a K4 expansion once the consumer's summed bits are set aside.
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
  if ((1 << kc) * (1 << dp->k) > (dp->dtype == QTN_C64 ? 32 : 16))
    return fail(QTN_E_UNSUPPORTED, "K6: %d B registers per thread", (1 << kc) * (1 << dp->k));
  int rc = make_plan(dp, 0, &F->p, smem, kc);
  if (rc) return rc;
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
      if (F->ng == MAXG) return fail(QTN_E_UNSUPPORTED, "K6: more than %d consumer members carry result bits", MAXG);
      const int g = F->ng++;
      F->gptr[g] = m.data;
      for (int j = 0; j < P.nH; ++j) F->ghs[g][j] = m.strides[P.hbit[j]];
      for (int t = 0; t < TBB; ++t) F->gtb[g][t] = (int32_t)m.strides[P.tbit[t]];
      for (int e = 0; e < P.nE; ++e) F->ge[g][e] = (int32_t)m.strides[P.ebit[e]];
      for (int q = 0; q < kc; ++q) F->gq[g][q] = (int32_t)m.strides[wc + q];
      F->gspan[g] = span;
    } else {
      const int u = F->nu++;
      F->uptr[u] = m.data;
      for (int q = 0; q < kc; ++q) F->uq[u][q] = (int32_t)m.strides[wc + q];
    }
  }
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
  *fn = dp->dtype == QTN_C64 ? fn_k6<float>(F->p.k, F->p.nq, F->p.nE) : fn_k6<double>(F->p.k, F->p.nq, F->p.nE);
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
