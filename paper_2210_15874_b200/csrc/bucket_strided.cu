// bucket_strided.cu — K3: one fused, permutation-aware bucket contraction.
//
// Replaces the reference's fast_kernel (src/tensor_core.py:148-164: transpose
// every member into [bucket, sorted result] order, broadcast-multiply into a
// (2,)*(w+1) buffer, sum axis 0) for a bucket whose members arrive in ANY
// axis order (standalone contract_bucket, the cfg-5 microbench).  No member
// is ever transposed in HBM: each is read once, coalesced, in its own order.
//
// Iteration space: result bits b = 0..w-1 (b = 0 the fastest axis of the
// sorted result, src/tensor_core.py:117-122) and the summed bit s = w.  Every
// member i has an element stride per iteration bit (0 = absent).
//
// Tiles.  The host picks T, a set of <= 12 result bits: the output's lowest
// bits first (coalesced stores), then, per large member, the result bits of
// its fastest axes until its contiguous run is >= 128 B, then more output
// bits up to the shared-memory budget.  A tile = 2^|T| results x both values
// of s.  Per tile every member's sub-tile (its bits in T u {s}, "local bits",
// in the member's own stride order) is staged in shared memory by cp.async
// (16-byte copies along stride-1 pairs), double-buffered across the
// persistent grid's tiles, so HBM reads are contiguous runs in the member's
// native order while the compute phase reads them in output order.
//
// Index maps are GF(2)-linear in the bits, so every offset is two 64-entry
// table lookups combined by add (global offsets) or xor (shared-memory slot).
// Shared-memory slots are XOR-swizzled per member so that the lanes of a
// half-warp (output bits 0..3) hit distinct banks in the compute phase while
// the staging phase (member bits 0..3) stays conflict-free too.
//
// out[r] = prod_i m_i(s=0, r) + prod_i m_i(s=1, r), members multiplied in
// bucket order (the reference's buf *= T_i, then buf.sum(axis=0)).
#include "qtn_b200.h"
#include "knobs.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

// error slot shared with qtn_b200.cu (qtn_last_error)
int qtn_internal_set_error(int code, const char* msg);

namespace qtn_k3 {

constexpr int NT = 256;
constexpr int MAXT = 12;              // tile bits
constexpr int MAXKS = 3;              // summed bits (one bucket index, or a merged chain of up to 3)
constexpr int MAXL = 14;              // local bits of a member (tile bits + summed bits <= 13)
constexpr int MAXM = QTN_MAX_MEMBERS;
constexpr int MAXN = QTN_MAX_WIDTH;   // non-tile result bits

struct Member {
  const void* ptr;
  int64_t nstride[MAXN];   // global stride of non-tile bit j of the tile id
  uint32_t lstride[MAXL];  // global stride of local bit q (ascending)
  uint16_t lphys[MAXL];    // shared-memory slot bits of local bit q (1<<q ^ swizzle)
  int8_t tq[MAXT];         // local bit of tile bit j, -1 if the member lacks it
  int8_t sq[MAXKS];        // local bit of summed bit i, -1 if the member lacks it
  int8_t nl;               // local bits
  int8_t vec;              // 2: stage stride-1 pairs with 16-byte copies (complex64)
  int32_t soff;            // element offset of the member's slots in a stage
  uint32_t fs[8];          // folded member: global stride of product-table bit b
  int64_t sstride[MAXKS];  // global stride of summed bit i (0 = absent)
};

struct Plan {
  void* out;
  int64_t onstride[MAXN];  // output stride of non-tile bit j (= 1 << bit)
  uint32_t otstride[MAXT]; // output stride of tile bit j
  int32_t w, nt, nn, nm;
  int32_t k;               // summed bits (iteration bits w .. w+k-1)
  int32_t stage_elems;     // elements of one stage (all members)
  int32_t table_bytes;
  int64_t n_tiles;
  // v2 (big/folded): members big[0..nb) are staged; members fold[0..nf) are
  // multiplied into a per-tile product table F over nu tile bits (fu) and s
  int32_t v2, nb, nf, nu;
  int8_t big[MAXM], fold[MAXM];
  int8_t fu[8];            // tile bit of table bit b
  int32_t f_off;           // byte offset of the two F buffers in dynamic smem
  int32_t bl_off;          // byte offset of the tile-base tables (v2)
  int32_t inv;             // v2: F (or big member 0) is the same for all of a thread's results
  unsigned long long* timing;   // program item timing (first start, last end), or null
  int32_t item;                 // program item id (timing slot)
  Member m[MAXM];
};

template <typename R> struct Cx;
template <> struct Cx<float> { using T = float2; };
template <> struct Cx<double> { using T = double2; };

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Loads from the dynamic shared memory at byte offsets: indexing the
// extern __shared__ array itself keeps the shared address space visible to
// the compiler (LDS [reg + imm], no generic-window arithmetic per access).
extern __shared__ __align__(16) unsigned char k3_dsmem[];
#ifndef K3_LDS_ASM
#define K3_LDS_ASM 1   // 0: C++ indexing (the compiler re-materialises the window base), 1: ld.shared
#endif
#if K3_LDS_ASM
// ld.shared at a 32-bit shared address (K3_LDS_ASM=2: with a memory clobber)
__device__ __forceinline__ uint32_t k3_smem_base() { return (uint32_t)__cvta_generic_to_shared(k3_dsmem); }
#if K3_LDS_ASM == 2
#define K3_CLOBBER : "memory"
#else
#define K3_CLOBBER
#endif
__device__ __forceinline__ float2 ld_sm(uint32_t a, float2*) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) K3_CLOBBER);
  return v;
}
__device__ __forceinline__ double2 ld_sm(uint32_t a, double2*) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) K3_CLOBBER);
  return v;
}
template <typename T>
__device__ __forceinline__ T lds(uint32_t off) {
  return ld_sm(off, static_cast<T*>(nullptr));
}
#else
__device__ __forceinline__ uint32_t k3_smem_base() { return 0u; }
template <typename T>
__device__ __forceinline__ T lds(uint32_t off) {
  return *reinterpret_cast<const T*>(k3_dsmem + off);
}
#endif

// Per-member lookup tables in shared memory (built once per block).
struct Tables {
  uint32_t GL[64], GH[128];  // global offset of local element e: GL[e & 63] + GH[e >> 6]
  uint16_t QL[64], QH[128];  // slot of local element e:          QL[e & 63] ^ QH[e >> 6]
  uint16_t PL[64], PH[64];   // slot of tile result r (s = 0):    PL[r & 63] ^ PH[r >> 6]
};

// tile id h -> element offset of the tile's first element for member x
// (x == NM: the output): lane j adds bit j of h times the stride of non-tile
// bit j, then a warp reduction; warp x % 8 handles x.  Strides are read from
// shared memory (copied once per block).
__device__ __forceinline__ void tile_bases(const int64_t (*ns)[MAXN], int nx, int nn, int64_t h, int64_t* dst) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int x = warp; x < nx; x += NT / 32) {
    int64_t o = 0;
    for (int j = lane; j < nn; j += 32)
      if ((h >> j) & 1) o += ns[x][j];
#pragma unroll
    for (int d = 16; d; d >>= 1) o += __shfl_xor_sync(0xffffffffu, o, d);
    if (lane == 0) dst[x] = o;
  }
}

// Stage the sub-tiles of members list[0..n) (tables tab[0..n)) of the tile
// whose bases are `base` (indexed by member) into stage `st`: one commit group.
template <typename R>
__device__ __forceinline__ void stage_tile(const Plan& P, const int8_t* list, int n_list, const Tables* tab,
                                           const int64_t* base, typename Cx<R>::T* st) {
  using T = typename Cx<R>::T;
  const int tid = threadIdx.x;
  for (int li = 0; li < n_list; ++li) {
    const int i = list ? list[li] : li;
    const Member& M = P.m[i];
    const T* src = reinterpret_cast<const T*>(M.ptr) + base[i];
    T* dst = st + M.soff;
    const Tables& tb = tab[li];
    const int n = 1 << M.nl;
    if (M.vec == 2) {
      for (int e = 2 * tid; e < n; e += 2 * NT) {
        const uint32_t g = tb.GL[e & 63] + tb.GH[e >> 6];
        const uint32_t q = tb.QL[e & 63] ^ tb.QH[e >> 6];
        cp_async16(dst + q, src + g);
      }
    } else {
      for (int e = tid; e < n; e += NT) {
        const uint32_t g = tb.GL[e & 63] + tb.GH[e >> 6];
        const uint32_t q = tb.QL[e & 63] ^ tb.QH[e >> 6];
        if (sizeof(T) == 16)
          cp_async16(dst + q, src + g);
        else
          cp_async8(dst + q, src + g);
      }
    }
  }
  cp_commit();
}

// Per-member lookup tables of one staged member (see Tables).
__device__ __forceinline__ void build_tables(const Plan& P, const Member& M, Tables& tb) {
  const int tid = threadIdx.x;
  for (int x = tid; x < 64 + 128; x += NT) {
    const int lo = x < 64;
    const int e = lo ? x : (x - 64) << 6;
    uint32_t g = 0, q = 0;
    for (int b = 0; b < M.nl; ++b)
      if ((e >> b) & 1) {
        g += M.lstride[b];
        q ^= M.lphys[b];
      }
    if (lo) {
      tb.GL[x] = g;
      tb.QL[x] = (uint16_t)q;
    } else {
      tb.GH[x - 64] = g;
      tb.QH[x - 64] = (uint16_t)q;
    }
  }
  for (int x = tid; x < 128; x += NT) {
    const int r = x < 64 ? x : (x - 64) << 6;
    uint32_t q = 0;
    for (int j = 0; j < P.nt; ++j)
      if (((r >> j) & 1) && M.tq[j] >= 0) q ^= M.lphys[M.tq[j]];
    if (x < 64)
      tb.PL[x] = (uint16_t)q;
    else
      tb.PH[x - 64] = (uint16_t)q;
  }
}

// Output offset of tile result r: OL[r & 63] + OH[r >> 6].
__device__ __forceinline__ void build_out_tables(const Plan& P, uint32_t* OL, uint32_t* OH) {
  for (int x = threadIdx.x; x < 128; x += NT) {
    const int r = x < 64 ? x : (x - 64) << 6;
    uint32_t o = 0;
    for (int j = 0; j < P.nt; ++j)
      if ((r >> j) & 1) o += P.otstride[j];
    if (x < 64)
      OL[x] = o;
    else
      OH[x - 64] = o;
  }
}

template <typename R, int NM>
__global__ void __launch_bounds__(NT) k3_kernel(const __grid_constant__ Plan P) {
  using T = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tables* tab = reinterpret_cast<Tables*>(smem_raw);
  uint32_t* OL = reinterpret_cast<uint32_t*>(smem_raw + NM * sizeof(Tables));
  uint32_t* OH = OL + 64;
  T* stage0 = reinterpret_cast<T*>(smem_raw + P.table_bytes);
  __shared__ int64_t sbase[3][NM + 1];   // ring of tile bases; [NM] = output
  __shared__ int64_t sns[NM + 1][MAXN];   // non-tile strides (members, output)
  const int tid = threadIdx.x;
  for (int x = tid; x < (NM + 1) * MAXN; x += NT) {
    const int i = x / MAXN, j = x % MAXN;
    sns[i][j] = i < NM ? P.m[i].nstride[j] : P.onstride[j];
  }

  // ---- tables ----
  for (int i = 0; i < NM; ++i) build_tables(P, P.m[i], tab[i]);
  build_out_tables(P, OL, OH);
  const int64_t G = gridDim.x;
  int64_t h = blockIdx.x;
  __syncthreads();
  // bases of the first two tiles (ring of 3: tile t uses slot t % 3)
  tile_bases(sns, NM + 1, P.nn, h, sbase[0]);
  if (h + G < P.n_tiles) tile_bases(sns, NM + 1, P.nn, h + G, sbase[1]);
  __syncthreads();
  if (h >= P.n_tiles) return;
  stage_tile<R>(P, nullptr, NM, tab, sbase[0], stage0);

  const int ntile = 1 << P.nt;
  const int rl = tid & 63;
  uint32_t pl[NM], ps[NM];
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    pl[i] = tab[i].PL[rl];
    ps[i] = P.m[i].lphys[P.m[i].sq[0]];
  }
  const uint32_t ol = OL[rl];
  int buf = 0, ring = 0;
  for (; h < P.n_tiles; h += G) {
    const int64_t hn = h + G;
    const int rn = ring == 2 ? 0 : ring + 1;
    if (hn < P.n_tiles) {
      stage_tile<R>(P, nullptr, NM, tab, sbase[rn], stage0 + (buf ^ 1) * P.stage_elems);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const T* st = stage0 + buf * P.stage_elems;
    T* out = reinterpret_cast<T*>(P.out) + sbase[ring][NM];
    const T* mb[NM];
#pragma unroll
    for (int i = 0; i < NM; ++i) mb[i] = st + P.m[i].soff;
#pragma unroll 2
    for (int r = tid; r < ntile; r += NT) {
      const int rh = r >> 6;
      T p0, p1;
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        const uint32_t q = pl[i] ^ tab[i].PH[rh];
        const T x0 = mb[i][q];
        const T x1 = mb[i][q ^ ps[i]];
        p0 = i == 0 ? x0 : cmul(p0, x0);
        p1 = i == 0 ? x1 : cmul(p1, x1);
      }
      __stcs(out + ol + OH[rh], cadd(p0, p1));
    }
    // bases of tile h + 2G into the ring slot tile h - G used
    const int64_t hnn = h + 2 * G;
    const int rnn = rn == 2 ? 0 : rn + 1;
    if (hnn < P.n_tiles) tile_bases(sns, NM + 1, P.nn, hnn, sbase[rnn]);
    __syncthreads();
    buf ^= 1;
    ring = rn;
  }
}

// ---------------------------------------------------------------------------
// v2: NB <= 4 staged ("big") members + the other (small, L1/L2-resident)
// members folded into a per-tile product table F[u][s] over the <= 5 tile
// bits they carry, so the per-result work is NB + 1 operands whatever the
// member count.  A thread owns results r = tid + j * NT (j < NJ): tile bits
// 0..7 come from tid, bits 8.. from j.  The planner picks those "j bits"
// among bits one operand (F, or big member 0) does not carry, so that
// operand is loaded once per tile (INV).  Every shared-memory offset a thread
// needs is tile-invariant and lives in registers; tile bases come from
// 3 x 7-bit lookup tables.
template <typename R, int MS>
__device__ __forceinline__ void compute_F(const Plan& P, const uint32_t* FG, const int64_t* base,
                                          typename Cx<R>::T* F) {
  using T = typename Cx<R>::T;
  const int k = MS ? P.k : 1;
  const int n = (1 << k) << P.nu;
  for (int x = threadIdx.x; x < n; x += NT) {
    const int u = x >> k;
    const int s = x & ((1 << k) - 1);
    // all loads in flight before the first multiply (members in order)
    T v[MAXM];
#pragma unroll
    for (int f = 0; f < MAXM; ++f) {
      if (f < P.nf) {
        const int i = P.fold[f];
        const Member& M = P.m[i];
        int64_t so = 0;
        if (MS) {
          for (int q = 0; q < k; ++q)
            if ((s >> q) & 1) so += M.sstride[q];
        } else if (s) {
          so = M.sstride[0];
        }
        const T* src = reinterpret_cast<const T*>(M.ptr) + base[i] + FG[f * 32 + (u & 15)] +
                       FG[f * 32 + 16 + (u >> 4)] + so;
        v[f] = __ldg(src);
      }
    }
    T prod = v[0];
#pragma unroll
    for (int f = 1; f < MAXM; ++f)
      if (f < P.nf) prod = cmul(prod, v[f]);
    F[x] = prod;
  }
}

// base of tile h for every member and the output (x = nm) from the 3-level
// tables BL[x][level][128]: one thread per entry
__device__ __forceinline__ void lut_bases(const int64_t* BL, int nx, int64_t h, int64_t* dst) {
  const int x = threadIdx.x;
  if (x < nx) {
    const int64_t* L = BL + x * 384;
    dst[x] = L[h & 127] + L[128 + ((h >> 7) & 127)] + L[256 + ((h >> 14) & 127)];
  }
}

template <typename R, int NB>
struct StageRegs {
  const typename Cx<R>::T* ptr[NB];
  uint32_t gl[NB], ql[NB];   // low-table entries of the thread's first element
  int n[NB], vec[NB];
  uint32_t dst[NB];          // byte offset of the member's slots in a stage
};

template <typename R, int NB>
__device__ __forceinline__ void stage_big(const Plan& P, const StageRegs<R, NB>& S, const Tables* tab,
                                          const int64_t* base, unsigned char* st) {
  using T = typename Cx<R>::T;
  const int tid = threadIdx.x;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const T* src = S.ptr[b] + base[P.big[b]];
    unsigned char* dst = st + S.dst[b];
    const int V = S.vec[b];
    const uint16_t* QH = tab[b].QH;
    const uint32_t* GH = tab[b].GH;
#pragma unroll 2
    for (int e = V * tid; e < S.n[b]; e += V * NT) {
      const int hi = e >> 6;
      const uint32_t g = S.gl[b] + GH[hi];
      const uint32_t q = (S.ql[b] ^ QH[hi]) * (uint32_t)sizeof(T);
      if (V == 2 || sizeof(T) == 16)
        cp_async16(dst + q, src + g);
      else
        cp_async8(dst + q, src + g);
    }
  }
  cp_commit();
}

template <typename R, int NB, int HF, int INV, int MS>
__global__ void __launch_bounds__(NT) k3v2_kernel(const __grid_constant__ Plan P) {
  using T = typename Cx<R>::T;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int NJ = sizeof(R) == 4 ? 8 : 4;
  // INV 1: F (or big member 0 when nothing is folded) is the same for all of a
  // thread's results; INV 2: F and big member 0 are (their product is hoisted)
  constexpr int B0 = (INV == 2 || (INV == 1 && !HF)) ? 1 : 0;   // first big member read per result
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tables* tab = reinterpret_cast<Tables*>(smem_raw);
  uint32_t* OL = reinterpret_cast<uint32_t*>(smem_raw + NB * sizeof(Tables));
  uint32_t* OH = OL + 64;
  uint32_t* FG = OH + 64;   // folded members: [f][16 low + 16 high] global offsets
  int64_t* BL = reinterpret_cast<int64_t*>(smem_raw + P.bl_off);
  unsigned char* stage0 = smem_raw + P.table_bytes;
  unsigned char* F0 = smem_raw + P.f_off;
  __shared__ int64_t sbase[3][MAXM + 1];
  const int tid = threadIdx.x;
  const int nm = P.nm;
  // ---- tables ----
#pragma unroll
  for (int b = 0; b < NB; ++b) build_tables(P, P.m[P.big[b]], tab[b]);
  build_out_tables(P, OL, OH);
  if (HF) {
    for (int x = tid; x < P.nf * 32; x += NT) {
      const Member& M = P.m[P.fold[x >> 5]];
      const int y = x & 31;
      const int u = y < 16 ? y : (y - 16) << 4;
      uint32_t g = 0;
      for (int b = 0; b < P.nu; ++b)
        if ((u >> b) & 1) g += M.fs[b];
      FG[x] = g;
    }
  }
  for (int x = tid; x < (nm + 1) * 384; x += NT) {
    const int i = x / 384, lv = (x % 384) >> 7, y = x & 127;
    const int64_t* ns = i < nm ? P.m[i].nstride : P.onstride;
    int64_t o = 0;
    for (int b = 0; b < 7; ++b) {
      const int j = lv * 7 + b;
      if (((y >> b) & 1) && j < P.nn) o += ns[j];
    }
    BL[x] = o;
  }
  const int64_t G = gridDim.x;
  int64_t h = blockIdx.x;
  __syncthreads();
  if (h >= P.n_tiles) return;
  // program graphs: inputs are predecessor outputs (PDL edge); standalone: no-op
  asm volatile("griddepcontrol.wait;" ::: "memory");
  unsigned long long t_start = 0;
  if (P.timing && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  lut_bases(BL, nm + 1, h, sbase[0]);
  if (h + G < P.n_tiles) lut_bases(BL, nm + 1, h + G, sbase[1]);
  StageRegs<R, NB> SR;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const Member& M = P.m[P.big[b]];
    SR.ptr[b] = reinterpret_cast<const T*>(M.ptr);
    SR.vec[b] = (M.vec == 2) ? 2 : 1;
    SR.n[b] = 1 << M.nl;
    SR.gl[b] = tab[b].GL[(SR.vec[b] * tid) & 63];
    SR.ql[b] = tab[b].QL[(SR.vec[b] * tid) & 63];
    SR.dst[b] = (uint32_t)M.soff * (uint32_t)sizeof(T);
  }
  __syncthreads();
  stage_big<R, NB>(P, SR, tab, sbase[0], stage0);
  const int fbytes = ((1 << P.k) << P.nu) * (int)sizeof(T);
  if (HF) compute_F<R, MS>(P, FG, sbase[0], reinterpret_cast<T*>(F0));

  // tile-invariant per-thread offsets (bytes into a stage / F buffer; elements of out)
  const int ntile = 1 << P.nt;
  const int nj = ntile >= NT ? ntile / NT : 1;
  uint32_t off[NB][NJ], offF[NJ], oo[NJ], psb[NB];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int r = (tid + j * NT) & (ntile - 1);
#pragma unroll
    for (int b = 0; b < NB; ++b)
      off[b][j] = ((uint32_t)(tab[b].PL[r & 63] ^ tab[b].PH[r >> 6]) + (uint32_t)P.m[P.big[b]].soff) * (uint32_t)sizeof(T);
    uint32_t u = 0;
    for (int b = 0; b < P.nu; ++b) u |= (uint32_t)((r >> P.fu[b]) & 1) << b;
    offF[j] = (u << P.k) * (uint32_t)sizeof(T);
    oo[j] = OL[r & 63] + OH[r >> 6];
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int8_t q0 = P.m[P.big[b]].sq[0];
    psb[b] = q0 >= 0 ? (uint32_t)P.m[P.big[b]].lphys[q0] * (uint32_t)sizeof(T) : 0u;
  }
  // multi-sum (MS): byte offset of each summed bit's plane per big member
  uint32_t sbit[NB][MAXKS];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int q = 0; q < MAXKS; ++q) {
      const int8_t sq = q < P.k ? P.m[P.big[b]].sq[q] : (int8_t)-1;
      sbit[b][q] = sq >= 0 ? (uint32_t)P.m[P.big[b]].lphys[sq] * (uint32_t)sizeof(T) : 0u;
    }
  const int NSr = 1 << P.k;
  const bool active = tid < ntile;
  const uint32_t stage_bytes = (uint32_t)P.stage_elems * (uint32_t)sizeof(T);

  int buf = 0, ring = 0;
  for (; h < P.n_tiles; h += G) {
    const int64_t hn = h + G;
    const int rn = ring == 2 ? 0 : ring + 1;
    if (hn < P.n_tiles) {
      stage_big<R, NB>(P, SR, tab, sbase[rn], stage0 + (buf ^ 1) * stage_bytes);
      if (HF) compute_F<R, MS>(P, FG, sbase[rn], reinterpret_cast<T*>(F0 + (buf ^ 1) * fbytes));
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const uint32_t stb = k3_smem_base() + (uint32_t)P.table_bytes + buf * stage_bytes;   // offsets into k3_dsmem
    const uint32_t Fb = k3_smem_base() + (uint32_t)P.f_off + buf * (uint32_t)fbytes;
    T* out = reinterpret_cast<T*>(P.out) + sbase[ring][nm];
    if (MS && active) {
      // summed assignments s = 0 .. 2^k - 1 outermost (ascending, as the
      // reference's bucket-by-bucket sums), a thread's NJ results inner
      T acc[NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[j] = T{};
      for (int s = 0; s < NSr; ++s) {
        uint32_t sp[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          uint32_t o = 0;
#pragma unroll
          for (int q = 0; q < MAXKS; ++q)
            if ((s >> q) & 1) o += sbit[b][q];
          sp[b] = stb + o;
        }
        T iv = T{};
        if (INV == 1) iv = HF ? lds<T>(Fb + offF[0] + s * (uint32_t)sizeof(T)) : lds<T>(sp[0] + off[0][0]);
        if (INV == 2) iv = cmul(lds<T>(Fb + offF[0] + s * (uint32_t)sizeof(T)), lds<T>(sp[0] + off[0][0]));
        auto term = [&](int j) {
          T p = iv;
#pragma unroll
          for (int b = B0; b < NB; ++b) {
            const T x = lds<T>(sp[b] + off[b][j]);
            p = (!INV && b == 0) ? x : cmul(p, x);
          }
          if (HF && INV == 0) p = cmul(p, lds<T>(Fb + offF[j] + s * (uint32_t)sizeof(T)));
          acc[j] = cadd(acc[j], p);   // acc starts at +0: s ascending, as the reference
        };
        if (nj == NJ) {
#pragma unroll
          for (int j = 0; j < NJ; ++j) term(j);
        } else {
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (j < nj) term(j);
        }
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        if (j < nj) __stcs(out + oo[j], acc[j]);
    }
    if (!MS && active) {
      T i0 = T{}, i1 = T{};
      if (INV == 1) {   // operand invariant across j: F, or big member 0
        if (HF) {
          i0 = lds<T>(Fb + offF[0]);
          i1 = lds<T>(Fb + offF[0] + (uint32_t)sizeof(T));
        } else {
          i0 = lds<T>(stb + off[0][0]);
          i1 = lds<T>(stb + off[0][0] + psb[0]);
        }
      }
      if (INV == 2) {   // F and big member 0 invariant: their product
        i0 = cmul(lds<T>(Fb + offF[0]), lds<T>(stb + off[0][0]));
        i1 = cmul(lds<T>(Fb + offF[0] + (uint32_t)sizeof(T)), lds<T>(stb + off[0][0] + psb[0]));
      }
      // per member: the s = 0 and s = 1 planes as two base addresses, so each
      // value is one shared load at [register offset + base]
      uint32_t s1p[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) s1p[b] = stb + psb[b];
      auto result = [&](int j) {
        T p0 = i0, p1 = i1;
#pragma unroll
        for (int b = B0; b < NB; ++b) {
          const T x0 = lds<T>(stb + off[b][j]);
          const T x1 = lds<T>(s1p[b] + off[b][j]);
          const bool first = !INV && b == 0;
          p0 = first ? x0 : cmul(p0, x0);
          p1 = first ? x1 : cmul(p1, x1);
        }
        if (HF && INV == 0) {
          p0 = cmul(p0, lds<T>(Fb + offF[j]));
          p1 = cmul(p1, lds<T>(Fb + offF[j] + (uint32_t)sizeof(T)));
        }
        __stcs(out + oo[j], cadd(p0, p1));
      };
      if (nj == NJ) {   // full tiles: no per-result guard
#pragma unroll
        for (int j = 0; j < NJ; ++j) result(j);
      } else {
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          if (j < nj) result(j);
      }
    }
    const int64_t hnn = h + 2 * G;
    const int rnn = rn == 2 ? 0 : rn + 1;
    if (hnn < P.n_tiles) lut_bases(BL, nm + 1, hnn, sbase[rnn]);
    __syncthreads();
    buf ^= 1;
    ring = rn;
  }
  if (P.timing && tid == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    atomicMin(&P.timing[2 * P.item], t_start);
    atomicMax(&P.timing[2 * P.item + 1], t_end);
  }
}

template <typename R, int NB, int HF, int MS>
const void* k3v2_fn_inv_ms(int inv) {
  if (HF && inv == 2) return (const void*)k3v2_kernel<R, NB, HF, (HF ? 2 : 1), MS>;
  return inv ? (const void*)k3v2_kernel<R, NB, HF, 1, MS> : (const void*)k3v2_kernel<R, NB, HF, 0, MS>;
}

template <typename R, int NB, int HF>
const void* k3v2_fn_inv(int inv, int ms) {
  return ms ? k3v2_fn_inv_ms<R, NB, HF, 1>(inv) : k3v2_fn_inv_ms<R, NB, HF, 0>(inv);
}

template <typename R>
const void* k3v2_fn(int nb, int hf, int inv, int ms) {
  switch (nb * 2 + (hf ? 1 : 0)) {
    case 2: return k3v2_fn_inv<R, 1, 0>(0, ms);
    case 3: return k3v2_fn_inv<R, 1, 1>(inv, ms);
    case 4: return k3v2_fn_inv<R, 2, 0>(inv, ms);
    case 5: return k3v2_fn_inv<R, 2, 1>(inv, ms);
    case 6: return k3v2_fn_inv<R, 3, 0>(inv, ms);
    case 7: return k3v2_fn_inv<R, 3, 1>(inv, ms);
    case 8: return k3v2_fn_inv<R, 4, 0>(inv, ms);
    case 9: return k3v2_fn_inv<R, 4, 1>(inv, ms);
    default: return nullptr;
  }
}

template <typename R>
const void* k3_fn(int nm) {
  switch (nm) {
    case 1: return (const void*)k3_kernel<R, 1>;
    case 2: return (const void*)k3_kernel<R, 2>;
    case 3: return (const void*)k3_kernel<R, 3>;
    case 4: return (const void*)k3_kernel<R, 4>;
    case 5: return (const void*)k3_kernel<R, 5>;
    case 6: return (const void*)k3_kernel<R, 6>;
    case 7: return (const void*)k3_kernel<R, 7>;
    case 8: return (const void*)k3_kernel<R, 8>;
    default: return nullptr;
  }
}

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return qtn_internal_set_error(code, buf);
}

// Host planner: tile bits, local bit orders, swizzles, shared-memory layout.
int make_plan(const qtn_bucket_desc_t* d, Plan* P, int* smem_bytes) {
  if (!d) return fail(QTN_E_INVALID, "null descriptor");
  if (d->dtype != QTN_C64 && d->dtype != QTN_C128) return fail(QTN_E_INVALID, "bad dtype %d", d->dtype);
  const int w = d->w, nm = d->n_mem;
  if (nm < 1 || nm > MAXM) return fail(QTN_E_INVALID, "bucket has %d members (1..%d)", nm, MAXM);
  if (w < 0 || w > 31) return fail(QTN_E_UNSUPPORTED, "result width %d outside 0..31", w);
  if (!d->out) return fail(QTN_E_INVALID, "null output");
  const int esz = d->dtype == QTN_C64 ? 8 : 16;
  const int BB = d->dtype == QTN_C64 ? 4 : 3;   // slot bits of one 128-byte bank row
  // summed bits: 1 (a reference bucket) or up to 3 (a merged chain, program items)
  const int ks = d->k > 0 ? d->k : 1;
  if (ks > MAXKS || w + ks > QTN_MAX_WIDTH + 1) return fail(QTN_E_UNSUPPORTED, "%d summed indices", ks);
  std::memset(P, 0, sizeof(*P));
  P->out = d->out;
  P->w = w;
  P->k = ks;
  P->nm = nm;
  int rank[MAXM];
  for (int i = 0; i < nm; ++i) {
    const qtn_bmember_t& m = d->mem[i];
    if (!m.data) return fail(QTN_E_INVALID, "member %d: null data", i);
    if (ks == 1 && m.strides[w] <= 0) return fail(QTN_E_INVALID, "member %d does not carry the bucket index", i);
    rank[i] = 0;
    for (int b = 0; b < w + ks; ++b) {
      if (m.strides[b] < 0) return fail(QTN_E_INVALID, "member %d: negative stride", i);
      if (m.strides[b]) ++rank[i];
    }
    if (rank[i] > 32) return fail(QTN_E_UNSUPPORTED, "member %d rank %d > 32", i, rank[i]);
    if (((uintptr_t)m.data) % esz) return fail(QTN_E_INVALID, "member %d misaligned", i);
  }
  if (((uintptr_t)d->out) % esz) return fail(QTN_E_INVALID, "output misaligned");

  // ---- tile bits ----
  // A thread owns results tid + j * NT: tile bits 0..7 ("core") come from
  // tid, bits 8.. ("j bits") from j < NJ = 8 (c64) / 4 (c128).
  const int tcap_env = qtn_knobs().k3_tcap;
  // local bits (tile + summed) stay <= 13: the staging tables are 6 + 7 bits
  const int tcap = std::min(std::min(d->dtype == QTN_C64 ? 11 : 10, 13 - ks), tcap_env > 0 ? tcap_env : 99);
  const int nt_target = std::min(tcap, w);
  const int core = std::min(nt_target, 8);
  bool inT[64] = {};
  int T[MAXT], nt = 0;
  bool staged[MAXM];
  for (int i = 0; i < nm; ++i) staged[i] = true;
  auto stage_elems = [&](int ntt) {   // elements of one stage if the tile bits were T[0..ntt)
    int64_t tot = 0;
    for (int i = 0; i < nm; ++i) {
      if (!staged[i]) continue;
      int nl = 0;
      for (int q = 0; q < ks; ++q)
        if (d->mem[i].strides[w + q]) ++nl;
      for (int j = 0; j < ntt; ++j)
        if (d->mem[i].strides[T[j]]) ++nl;
      tot += ((int64_t)1 << nl) + 1;   // +1: 16-byte aligned member slots
    }
    return tot;
  };
  const int budget_kb = qtn_knobs().k3_stage_kb;
  const int64_t budget = (budget_kb * 1024) / esz;   // one stage; two are resident
  auto add = [&](int b, bool check) {
    if (b >= w || inT[b] || nt >= tcap) return false;
    T[nt++] = b;
    if (check && stage_elems(nt) > budget) {
      --nt;
      return false;
    }
    inT[b] = true;
    return true;
  };
  for (int b = 0; b < std::min(w, 5); ++b) add(b, false);   // coalesced 32-lane stores
  // per member (largest first): its fastest axes until a >= 128-byte run
  int ord[MAXM];
  for (int i = 0; i < nm; ++i) ord[i] = i;
  std::stable_sort(ord, ord + nm, [&](int a, int b) { return rank[a] > rank[b]; });
  const int run_bytes = qtn_knobs().k3_run;
  const int64_t run_target = std::max(1, run_bytes / esz);
  for (int oi = 0; oi < nm; ++oi) {
    const qtn_bmember_t& m = d->mem[ord[oi]];
    if (rank[ord[oi]] < 3) continue;
    int64_t run = 1;
    while (run < run_target && nt < core) {
      int b = -1;   // the axis with stride == run
      for (int c = 0; c < w + ks; ++c)
        if (m.strides[c] == run) b = c;
      if (b < 0) break;
      if (b < w && !inT[b] && !add(b, true)) break;
      run *= 2;
    }
  }
  auto member_tbits = [&](int i) {
    uint32_t t = 0;
    for (int j = 0; j < nt; ++j)
      if (d->mem[i].strides[T[j]]) t |= 1u << j;
    return t;
  };
  // fold small (L1/L2-resident) members while their tile bits stay <= ulim
  int imax = 0;
  for (int i = 1; i < nm; ++i)
    if (__builtin_popcount(member_tbits(i)) > __builtin_popcount(member_tbits(imax))) imax = i;
  bool folded[MAXM] = {};
  const bool v2_off = qtn_knobs().k3_v1 != 0;
  if (!v2_off) {
    int cand[MAXM], nc = 0;
    for (int i = 0; i < nm; ++i)
      if (i != imax && rank[i] <= 12) cand[nc++] = i;
    std::stable_sort(cand, cand + nc,
                     [&](int a, int b) { return __builtin_popcount(member_tbits(a)) < __builtin_popcount(member_tbits(b)); });
    const int ulim_env = qtn_knobs().k3_ulim;
    const int ulim = std::min(ulim_env, std::max(0, core - 2));
    uint32_t U = 0;
    for (int c = 0; c < nc; ++c) {
      const uint32_t U2 = U | member_tbits(cand[c]);
      if (__builtin_popcount(U2) <= ulim) {
        U = U2;
        folded[cand[c]] = true;
        staged[cand[c]] = false;
      }
    }
  }
  int nb = 0, nf = 0;
  for (int i = 0; i < nm; ++i) nb += folded[i] ? 0 : 1, nf += folded[i] ? 1 : 0;
  P->v2 = (nb <= 4 && !v2_off) ? 1 : 0;
  if (!P->v2 && ks > 1) return fail(QTN_E_UNSUPPORTED, "%d staged members with %d summed indices", nb, ks);
  if (!P->v2) {
    for (int i = 0; i < nm; ++i) folded[i] = false, staged[i] = true;
    nf = 0;
    nb = nm;
  }
  // the invariant operand: F if any member is folded, else the staged member
  // with the fewest indices (when there are two or more); the j bits avoid
  // every index it carries
  int inv_member = -1;
  bool has_inv = false;
  uint64_t avoid = 0;     // iteration bits of the invariant operands
  uint64_t avoid_f = 0;   // ... of the folded table F alone
  auto member_bits = [&](int i) {
    uint64_t a = 0;
    for (int b = 0; b < w; ++b)
      if (d->mem[i].strides[b]) a |= 1ull << b;
    return a;
  };
  int inv_cand = -1;   // staged member with the fewest indices (never the widest)
  for (int i = 0; i < nm; ++i)
    if (!folded[i] && i != imax && (inv_cand < 0 || rank[i] < rank[inv_cand])) inv_cand = i;
  if (P->v2 && nf > 0) {
    has_inv = true;
    for (int i = 0; i < nm; ++i)
      if (folded[i]) avoid_f |= member_bits(i);
    avoid = avoid_f;
    // level 2: F and one staged member invariant, when enough bits remain for j
    const bool inv2_off = qtn_knobs().k3_inv2 == 0;
    if (!inv2_off && nb >= 2 && inv_cand >= 0) {
      const uint64_t a2 = avoid_f | member_bits(inv_cand);
      int free_bits = 0;
      for (int b = 0; b < w; ++b)
        if (!inT[b] && !((a2 >> b) & 1)) ++free_bits;
      if (free_bits >= nt_target - core) {   // only with full-size tiles
        inv_member = inv_cand;
        avoid = a2;
      }
    }
  } else if (P->v2 && nb >= 2) {
    inv_member = inv_cand;
    has_inv = true;
    avoid = member_bits(inv_member);
  }
  // j bits: the lowest bits the invariant operand lacks, reserved first; the
  // core is filled with the invariant operand's own bits first when it is a
  // staged member (free), last when it is F (they would grow the table)
  int nt_goal = nt_target;
  {
    int jres[4], nj_res = 0;
    for (int b = 0; b < w && nj_res < nt_target - core; ++b)
      if (!inT[b] && !((avoid >> b) & 1)) jres[nj_res++] = b;
    // too few: a smaller tile that keeps the operand invariant (>= 4 results/thread)
    if (has_inv && nj_res < nt_target - core && nj_res >= 2) nt_goal = core + nj_res;
    auto reserved = [&](int b) {
      for (int q = 0; q < nj_res; ++q)
        if (jres[q] == b) return true;
      return false;
    };
    // core fill: bits of an invariant staged member first (free), then bits
    // no invariant operand carries, F's bits last (they would grow the table)
    const uint64_t avoid_big = avoid & ~avoid_f;
    for (int pass = 0; pass < 4 && nt < core; ++pass)
      for (int b = 0; b < w && nt < core; ++b) {
        if (inT[b]) continue;
        const bool ok = pass == 3   ? true
                        : pass == 0 ? (((avoid_big >> b) & 1) && !reserved(b))
                        : pass == 1 ? (!((avoid >> b) & 1) && !reserved(b))
                                    : !reserved(b);
        if (ok && !add(b, true)) pass = 4, b = w;
      }
    for (int q = 0; q < nj_res && nt < nt_goal; ++q)
      if (!inT[jres[q]] && !add(jres[q], true)) break;
    for (int b = 0; b < w && nt < nt_goal; ++b)
      if (!inT[b] && !add(b, true)) break;
  }
  bool inv_f = has_inv, inv_b = inv_member >= 0;
  for (int j = 8; j < nt; ++j) {
    if (((nf > 0 ? avoid_f : 0) >> T[j]) & 1) inv_f = false;
    if (inv_member >= 0 && ((member_bits(inv_member) >> T[j]) & 1)) inv_b = false;
  }
  // INV 1: F (or, with no folded member, big member 0) invariant; 2: F and big member 0
  if (nf > 0)
    P->inv = inv_f ? (inv_b ? 2 : 1) : 0;
  else
    P->inv = inv_b ? 1 : 0;

  P->nt = nt;
  int N[MAXN], nn = 0;
  for (int b = 0; b < w; ++b)
    if (!inT[b]) N[nn++] = b;
  if (nn > 21) return fail(QTN_E_UNSUPPORTED, "%d non-tile bits > 21", nn);
  P->nn = nn;
  P->n_tiles = (int64_t)1 << nn;
  for (int j = 0; j < nt; ++j) P->otstride[j] = 1u << T[j];
  for (int j = 0; j < nn; ++j) P->onstride[j] = (int64_t)1 << N[j];

  // ---- member roles ----
  const bool inv_big = P->v2 && inv_member >= 0 && ((nf == 0 && P->inv == 1) || P->inv == 2);   // big member 0 invariant
  nb = nf = 0;
  if (inv_big) P->big[nb++] = (int8_t)inv_member;
  for (int i = 0; i < nm; ++i) {
    if (folded[i])
      P->fold[nf++] = (int8_t)i;
    else if (!(inv_big && i == inv_member))
      P->big[nb++] = (int8_t)i;
  }
  P->nb = nb;
  P->nf = nf;
  P->nu = 0;
  for (int j = 0; j < nt; ++j) {
    bool any = false;
    for (int f = 0; f < nf; ++f)
      if (d->mem[P->fold[f]].strides[T[j]]) any = true;
    if (any) P->fu[P->nu++] = (int8_t)j;
  }
  if (P->nu > 8) return fail(QTN_E_UNSUPPORTED, "product table of %d bits", P->nu);

  int64_t soff = 0;
  for (int i = 0; i < nm; ++i) {
    const qtn_bmember_t& m = d->mem[i];
    Member& M = P->m[i];
    M.ptr = m.data;
    for (int q = 0; q < MAXKS; ++q) {
      M.sstride[q] = q < ks ? m.strides[w + q] : 0;
      M.sq[q] = -1;
    }
    for (int j = 0; j < nn; ++j) M.nstride[j] = m.strides[N[j]];
    for (int b = 0; b < P->nu; ++b) M.fs[b] = (uint32_t)m.strides[T[P->fu[b]]];
    // local bits: the member's bits in T u {summed bits}, ascending stride
    int lb[MAXL], nl = 0;   // iteration bit of local bit q (>= w: summed)
    for (int j = 0; j < nt; ++j)
      if (m.strides[T[j]]) lb[nl++] = T[j];
    for (int q = 0; q < ks; ++q)
      if (m.strides[w + q]) lb[nl++] = w + q;
    std::sort(lb, lb + nl, [&](int a, int b) { return m.strides[a] < m.strides[b]; });
    M.nl = (int8_t)nl;
    for (int q = 0; q < nl; ++q) M.lstride[q] = (uint32_t)m.strides[lb[q]];
    for (int j = 0; j < nt; ++j) M.tq[j] = -1;
    uint32_t smask_local = 0;   // local bits of summed indices (never swizzle targets)
    for (int q = 0; q < nl; ++q) {
      if (lb[q] >= w) {
        M.sq[lb[q] - w] = (int8_t)q;
        smask_local |= 1u << q;
      } else {
        for (int j = 0; j < nt; ++j)
          if (T[j] == lb[q]) M.tq[j] = (int8_t)q;
      }
    }
    bool vec2 = nl > 0 && esz == 8 && m.strides[lb[0]] == 1 && ((uintptr_t)m.data % 16) == 0;
    for (int b = 0; b < w + ks; ++b)
      if (b != lb[0] && (m.strides[b] & 1)) vec2 = false;   // pairs stay 16-byte aligned
    M.vec = vec2 ? 2 : 1;
    // swizzle: local bits q >= BB that the compute-phase half-warp varies
    // (tile bits 0..BB-1) get a distinct free low slot bit; never the slot
    // bit of s (the s = 1 value stays at a constant additive offset) and, for
    // 16-byte staging, never slot bit 0
    uint32_t span = 0;
    const int lo_ok = vec2 ? 1 : 0;
    for (int q = 0; q < nl; ++q) M.lphys[q] = (uint16_t)(1u << q);
    for (int j = 0; j < std::min(BB, nt); ++j)
      if (M.tq[j] >= 0 && M.tq[j] < BB) span |= 1u << M.tq[j];
    for (int j = 0; j < std::min(BB, nt); ++j) {
      const int q = M.tq[j];
      if (q < BB) continue;
      for (int b = lo_ok; b < BB; ++b)
        if (!((smask_local >> b) & 1) && !((span >> b) & 1)) {
          span |= 1u << b;
          M.lphys[q] ^= (uint16_t)(1u << b);
          break;
        }
    }
    if (folded[i]) continue;   // not staged
    const int64_t n = (int64_t)1 << nl;
    soff = (soff + 1) & ~(int64_t)1;   // 16-byte aligned slots (complex64)
    M.soff = (int32_t)soff;
    soff += n;
  }
  soff = (soff + 1) & ~(int64_t)1;
  P->stage_elems = (int32_t)soff;
  const int ntab = P->v2 ? nb : nm;
  P->table_bytes = (int32_t)(((int64_t)ntab * sizeof(Tables) + 128 * 4 + (int64_t)nf * 32 * 4 + 15) / 16 * 16);
  P->f_off = P->table_bytes + 2 * P->stage_elems * esz;
  P->bl_off = P->f_off + (nf ? 2 * ((1 << ks) << P->nu) * esz : 0);
  *smem_bytes = P->bl_off + (P->v2 ? (nm + 1) * 384 * 8 : 0);
  if (*smem_bytes > 227 * 1024) return fail(QTN_E_UNSUPPORTED, "bucket needs %d B of shared memory", *smem_bytes);
  return QTN_OK;
}

int sm_count() {
  int dev = 0, nsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return nsm;
}

}  // namespace qtn_k3

// Program-graph node for one item (called by qtn_graph_create, qtn_b200.cu):
// plans K3 for `d` into `plan` (size qtn_k3_plan_bytes()) and returns the
// kernel, grid and dynamic shared memory.
size_t qtn_k3_plan_bytes() { return sizeof(qtn_k3::Plan); }

int qtn_k3_node(const qtn_bucket_desc_t* d, unsigned long long* timing, int32_t item, void* plan, const void** fn,
                int* grid, int* smem) {
  using namespace qtn_k3;
  Plan* P = reinterpret_cast<Plan*>(plan);
  int rc = make_plan(d, P, smem);
  if (rc) return rc;
  if (!P->v2) return fail(QTN_E_UNSUPPORTED, "K3 node needs the staged/folded kernel");
  P->timing = timing;
  P->item = item;
  *fn = d->dtype == QTN_C64 ? k3v2_fn<float>(P->nb, P->nf > 0, P->inv, P->k > 1)
                            : k3v2_fn<double>(P->nb, P->nf > 0, P->inv, P->k > 1);
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
  if (per_sm < 1) return fail(QTN_E_UNSUPPORTED, "K3 cannot be resident with %d B smem", *smem);
  *grid = (int)std::min<int64_t>(P->n_tiles, (int64_t)per_sm * sm_count());
  return QTN_OK;
}

extern "C" {

int qtn_bucket_plan(const qtn_bucket_desc_t* d, int32_t* info) {
  using namespace qtn_k3;
  static thread_local Plan P;
  int smem = 0;
  const int rc = make_plan(d, &P, &smem);
  if (rc) return rc;
  if (info) {
    info[0] = P.nt;
    info[1] = P.stage_elems;
    info[2] = smem;
    info[3] = (int32_t)std::min<int64_t>(P.n_tiles, INT32_MAX);
    info[4] = P.v2 ? P.nb : -1;
    info[5] = P.nf;
    info[6] = P.nu;
    info[7] = P.inv;
  }
  return QTN_OK;
}

int qtn_bucket(const qtn_bucket_desc_t* d, void* stream) {
  using namespace qtn_k3;
  static thread_local Plan P;
  int smem = 0;
  int rc = make_plan(d, &P, &smem);
  if (rc) return rc;
  const void* fn = P.v2 ? (d->dtype == QTN_C64 ? k3v2_fn<float>(P.nb, P.nf > 0, P.inv, P.k > 1)
                                                : k3v2_fn<double>(P.nb, P.nf > 0, P.inv, P.k > 1))
                       : (d->dtype == QTN_C64 ? k3_fn<float>(P.nm) : k3_fn<double>(P.nm));
  cudaFuncAttributes fa;   // the attribute only grows (graph nodes of the same kernel may need more)
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return fail(QTN_E_CUDA, "cudaFuncGetAttributes: %s", cudaGetErrorString(e));
  if (smem > fa.maxDynamicSharedSizeBytes) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return fail(QTN_E_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem);
  if (e != cudaSuccess) return fail(QTN_E_CUDA, "occupancy: %s", cudaGetErrorString(e));
  if (per_sm < 1) return fail(QTN_E_UNSUPPORTED, "K3 cannot be resident with %d B smem", smem);
  const int64_t grid = std::min<int64_t>(P.n_tiles, (int64_t)per_sm * sm_count());
  void* args[] = {&P};
  e = cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(NT), args, smem, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(QTN_E_CUDA, "K3 launch: %s", cudaGetErrorString(e));
  return QTN_OK;
}

}  // extern "C"
