// qtn_b200.cu — sm_100a kernels + C ABI of the bucket-elimination engine.
//
// A planned program (engine.py) is a list of *items* — one reference bucket
// (src/ordering.py:175-187), or a chain of them merged into one contraction
// summing k indices — in a topological order, grouped into graph *nodes*:
//
//  K2  small_kernel   A persistent launch over a stage of small items (result
//      tiles below one vector step).  Tickets are stage-relative; a block that
//      takes a ticket only waits on LOWER tickets of the same stage (per-item
//      completion counters, acquire/release), so the schedule is deadlock-free
//      whatever the residency.  Threads cover (result element, summed
//      assignment) pairs, read members straight from L2 and reduce the
//      assignments in order through shared memory.  Finaliser items multiply
//      an instance's rank-0 values into its result slot (get-result,
//      src/ordering.py:167-170,183-184).
//
//  K1  large_kernel   One launch per large item, specialised at compile time
//      by (NS = 2^k, NV = varying staged members, ST = one streamed member),
//      so every variant gets its own register allocation.  A tile is 2^L
//      consecutive results; members are classified by the planner:
//        streamed   carries every tile bit — 16-byte loads from HBM/L2, the NS
//                   summed-assignment values prefetched together
//        uniform    carries no tile bit — folded into U[s] once per tile
//        invariant  carries none of the thread's step bits — folded into P[s]
//                   in registers once per tile (k == 1)
//        varying    staged in shared memory by bulk async copies (TMA engine,
//                   cp.async.bulk + mbarrier), gathered per step
//      out[r] = sum_s prod_i member_i(s, r), s ascending (deterministic).
//
// Nodes are stitched into one CUDA graph per program (dependency edges from
// the item DAG), so independent items overlap and a whole lightcone is one
// cudaGraphLaunch.  Data produced inside a launch by other blocks is read with
// ld.global.cg (L2) — never a stale L1 line.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo ...
#include "qtn_b200.h"
#include "knobs.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_err(cudaError_t e, const char* what) {
  return set_err(QTN_E_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// QTN_DEBUG build: bounds-check every arena / shared-memory index (trap with
// a message).  compute-sanitizer is unavailable on the target pool.
#ifdef QTN_DEBUG
#define QTN_CHECK(cond, ...)                                                     \
  do {                                                                           \
    if (!(cond)) {                                                               \
      printf("QTN_CHECK %s:%d (block %d thread %d): ", __FILE__, __LINE__,      \
             (int)blockIdx.x, (int)threadIdx.x);                                \
      printf(__VA_ARGS__);                                                       \
      printf("\n");                                                             \
      __trap();                                                                  \
    }                                                                            \
  } while (0)
#else
#define QTN_CHECK(cond, ...) \
  do {                       \
  } while (0)
#endif
#define QTN_ARENA_OK(P, o) ((P).arena_elems == 0 || ((int64_t)(o) >= 0 && (int64_t)(o) < (P).arena_elems))

constexpr int NT = 256;                 // threads per block

constexpr int MAXM = QTN_MAX_MEMBERS;   // members per item
constexpr int MAXS = 16;                // vector steps per tile: 2^L / (VEC * NT)
constexpr int MAXNS = 1 << QTN_MAX_SUMMED;
constexpr int SMALL_PROD_ELEMS = 1024;  // smem products per round of a small tile
constexpr int K2_HI_SLOT = 64;          // staged double-precision input member (rank <= 6)

template <typename R> struct Cx;
template <> struct Cx<float> {
  using T = float2;   // one complex64
  using V = float4;   // two consecutive complex64 (16 B)
  static constexpr int VEC = 2;
};
template <> struct Cx<double> {
  using T = double2;  // one complex128 (16 B)
  using V = double2;
  static constexpr int VEC = 1;
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

__device__ __forceinline__ double2 widen(float2 a) { return make_double2((double)a.x, (double)a.y); }
__device__ __forceinline__ double2 widen(double2 a) { return a; }
__device__ __forceinline__ void narrow(double2 a, float2& o) { o = make_float2((float)a.x, (float)a.y); }
__device__ __forceinline__ void narrow(double2 a, double2& o) { o = a; }

__device__ __forceinline__ void split(float4 v, float2 (&e)[2]) {
  e[0] = make_float2(v.x, v.y);
  e[1] = make_float2(v.z, v.w);
}
__device__ __forceinline__ void split(double2 v, double2 (&e)[1]) { e[0] = v; }
__device__ __forceinline__ float4 join(const float2 (&e)[2]) { return make_float4(e[0].x, e[0].y, e[1].x, e[1].y); }
__device__ __forceinline__ double2 join(const double2 (&e)[1]) { return e[0]; }

__device__ __forceinline__ uint32_t pext32(uint32_t x, uint32_t m) {
  uint32_t r = 0;
  for (int k = 0; m; ++k) {
    const uint32_t low = m & (0u - m);
    if (x & low) r |= 1u << k;
    m ^= low;
  }
  return r;
}
__device__ __forceinline__ uint32_t pdep32(uint32_t x, uint32_t m) {
  uint32_t r = 0;
  for (int k = 0; m; ++k) {
    const uint32_t low = m & (0u - m);
    if ((x >> k) & 1u) r |= low;
    m ^= low;
  }
  return r;
}
__device__ __forceinline__ uint64_t pext64(uint64_t x, uint64_t m) {
  uint64_t r = 0;
  for (int k = 0; m; ++k) {
    const uint64_t low = m & (0ull - m);
    if (x & low) r |= 1ull << k;
    m ^= low;
  }
  return r;
}

#ifndef K2_RED_RELEASE
#define K2_RED_RELEASE 1
#endif
// Publish n finished tiles of an item (thread 0, after a __syncthreads that
// ordered the block's result stores): one release-add at gpu scope, the
// consumer's ld.acquire pairs with it (cumulativity covers the other
// threads' stores via the barrier).
__device__ __forceinline__ void publish_tiles(uint32_t* p, uint32_t n) {
#if K2_RED_RELEASE
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(n) : "memory");
#else
  __threadfence();
  atomicAdd(p, n);
#endif
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Programmatic dependent launch (PDL): a kernel lets its graph successors
// launch as soon as all of its blocks are running, and a successor waits for
// its predecessors' completion (and memory) only where it first reads their
// outputs — launch latency and table prologues overlap the predecessor.
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// K2 stages warm L2 with their item / member records and the input image
#ifndef K2_WARM
#define K2_WARM 1
#endif
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

[[maybe_unused]] __device__ __forceinline__ uint32_t dyn_smem_bytes() {
  uint32_t v;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- mbarrier + bulk async copy (TMA engine, non-tensor form) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

// =========================================================================
// K2: persistent small-stage kernel
// =========================================================================
struct SmallCtx {
  qtn_bucket_t b;
  uint64_t base[MAXM];
  uint64_t mhi[MAXM];
  uint64_t off[MAXM];
  uint32_t mlo[MAXM];
  int32_t pc[MAXM];
  int32_t pclo[MAXM];
  int16_t sig[MAXM][MAXNS];
  int32_t hmode[MAXM];   // 1: input member staged unrounded in shi (complex64 programs, rank <= 6)
  int32_t item;
  int32_t tick;
  int32_t next;
  int32_t last;
  int32_t item_end;   // first ticket after the current item
};

template <typename R>
__global__ void __launch_bounds__(NT) small_kernel(const qtn_program_t P, int32_t first, int32_t count,
                                                   int32_t n_tickets, uint32_t* ctl, uint32_t jitter) {
  using T = typename Cx<R>::T;
  // complex64 programs may carry unrounded inputs (P.inputs_hi), staged in
  // shared memory as complex128 before the item waits for its producers
  // (complex128 programs read their inputs in the compute loop: staging them
  // too measured 12 % slower on cfg-2)
  constexpr bool HI = Cx<R>::VEC == 2;
  // K2 computes in double at both element types: products and the in-order
  // sum over assignments are rounded once, when the result is stored; input
  // members of complex64 programs come unrounded from P.inputs_hi
  using D = double2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  D* sprod = reinterpret_cast<D*>(smem_raw);
  __shared__ SmallCtx S;
  // unrounded input members of the current item (complex64 programs), one
  // slot of K2_HI_SLOT elements per member
  double2* shi = reinterpret_cast<double2*>(smem_raw + SMALL_PROD_ELEMS * sizeof(D));
  const T* A = reinterpret_cast<const T*>(P.arena);
  T* Aw = reinterpret_cast<T*>(P.arena);
  const double2* Ahi = reinterpret_cast<const double2*>(P.inputs_hi);
  const uint64_t n_hi = (HI && Ahi) ? (uint64_t)P.n_in_elems : 0ull;
  uint32_t* done = P.ctrl + 2 * P.n_nodes;
  const int tid = threadIdx.x;
  const int last_item = first + count - 1;
  int cur = first;
  int prepared = -1;
  uint32_t pend_cnt = 0;   // thread 0: finished, unpublished tiles of pend_item
  int pend_item = 0;

  pdl_launch_dependents();
#if K2_WARM
  // Warm L2 with what every item of the stage reads first: the stage's item
  // and member records and the program's input image (cold after an L2
  // flush or between calls).  L2 is the coherence point, so lines a
  // predecessor node is still writing stay correct.
  {
    const size_t stride = (size_t)gridDim.x * NT * 128;
    const size_t t0 = ((size_t)blockIdx.x * NT + tid) * 128;
    const char* b0 = reinterpret_cast<const char*>(P.buckets + first);
    for (size_t o = t0; o < (size_t)count * sizeof(qtn_bucket_t); o += stride) prefetch_l2(b0 + o);
    const size_t ib = (size_t)P.n_in_elems * sizeof(T);
    for (size_t o = t0; o < ib; o += stride) prefetch_l2(reinterpret_cast<const char*>(P.arena) + o);
    if (HI && P.inputs_hi)
      for (size_t o = t0; o < (size_t)P.n_in_elems * 16; o += stride)
        prefetch_l2(reinterpret_cast<const char*>(P.inputs_hi) + o);
    if (blockIdx.x == 0 && tid < 32) {
      const int m0 = __ldg(&P.buckets[first].mem_begin);
      const int m1 = __ldg(&P.buckets[first + count - 1].mem_begin) + 8;
      const char* mb = reinterpret_cast<const char*>(P.members + m0);
      for (size_t o = (size_t)tid * 128; o < (size_t)(m1 - m0) * sizeof(qtn_member_t); o += 32 * 128)
        prefetch_l2(mb + o);
    }
  }
#endif
  // The stage's counters were zeroed by its previous run's last block (or by
  // qtn_program_reset), both stream-ordered before this graph launch, and the
  // program records are uploaded before it: the first ticket, its search and
  // the item's records are fetched BEFORE waiting for the predecessor nodes
  // (griddepcontrol.wait below, ahead of the first read of data a node writes)
  bool waited = false;
  if (tid == 0) S.next = (int)atomicAdd(&ctl[0], 1u);
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      S.tick = S.next;
      if (S.tick < n_tickets) S.next = (int)atomicAdd(&ctl[0], 1u);   // prefetch
    }
    __syncthreads();
    const int tk = S.tick;
    if (tk >= n_tickets) break;
    // ---- ticket -> item: 32-ary search over tick_begin[cur..last] (warp 0) ----
    if (tid < 32) {
      int lo = cur, hi = last_item;
      if (lo < hi && __ldg(&P.tick_begin[lo + 1]) > tk) hi = lo;
      while (hi > lo) {
        const int step = (hi - lo + 31) / 32;
        int p = lo + (tid + 1) * step;
        if (p > hi) p = hi;
        const unsigned bal = __ballot_sync(0xffffffffu, __ldg(&P.tick_begin[p]) <= tk);
        const int c = __popc(bal);
        if (c == 0) {
          hi = lo + step - 1;
        } else {
          const int plast = min(lo + c * step, hi);
          const int pnext = lo + (c + 1) * step;
          lo = plast;
          if (c < 32 && pnext - 1 < hi) hi = pnext - 1;
        }
      }
      if (tid == 0) {
        S.item = lo;
        if (lo != prepared) {
          S.b = P.buckets[lo];
          S.item_end = lo < last_item ? __ldg(&P.tick_begin[lo + 1]) : n_tickets;
        }
      }
    }
    __syncthreads();
    cur = S.item;
    if (cur != prepared) {
      // publish finished tiles of the previous item before any waiting
      if (tid == 0 && pend_cnt) {
        publish_tiles(&done[pend_item], pend_cnt);
        pend_cnt = 0;
      }
      const int nm = S.b.w >= 0 ? S.b.n_mem : 0;
      const int L = S.b.tile_bits;
      const int k = S.b.w >= 0 ? S.b.k : 0;
      if (tid < nm) {
        const qtn_member_t m = P.members[S.b.mem_begin + tid];
        const uint32_t lowmask = (1u << L) - 1u;
        S.off[tid] = m.off;
        S.mlo[tid] = (uint32_t)(m.mask & lowmask);
        S.mhi[tid] = m.mask >> L;
        S.pc[tid] = __popcll(m.mask);
        S.pclo[tid] = __popc((uint32_t)(m.mask & lowmask));
        for (int q = 0; q < (1 << k); ++q) S.sig[tid][q] = (int16_t)pext32((uint32_t)q, m.smask);
        const int lg = __popcll(m.mask) + __popc(m.smask);
        S.hmode[tid] = (HI && m.off < n_hi && lg <= 6) ? 1 : 0;
      }
      if (!waited) {
        pdl_wait();   // predecessor nodes' outputs visible
        waited = true;
      }
      if (HI && n_hi) {
        // stage the item's (small) input members unrounded
        for (int e = tid; e < nm * K2_HI_SLOT; e += NT) {
          const qtn_member_t m = P.members[S.b.mem_begin + e / K2_HI_SLOT];
          const int q = e % K2_HI_SLOT;
          const int lg = __popcll(m.mask) + __popc(m.smask);
          if (HI && m.off < n_hi && lg <= 6 && q < (1 << lg)) shi[e] = __ldg(Ahi + m.off + q);
        }
      }
#ifndef QTN_MUTANT_NO_WAIT   // mutation build (make variant EXTRA=-DQTN_MUTANT_NO_WAIT): proves the race test bites
      for (int d = tid; d < S.b.n_dep; d += NT) {
#else
      for (int d = tid; d < 0; d += NT) {
#endif
        const qtn_dep_t dp = P.deps[S.b.dep_begin + d];
        const uint32_t* c = done + dp.bucket;
        int spins = 0;
        while (ld_acquire(c) < (uint32_t)dp.need) {
          if (++spins > 64) __nanosleep(32);
        }
      }
      __syncthreads();
      prepared = cur;
    }
    const int h = tk - S.b.tick_begin;
    if (jitter) {
      // schedule perturbation (QTN_K2_JITTER, race tests): the block stalls a
      // pseudo-random 0-4 us before computing the tile, so producers finish
      // in an order unrelated to their tickets; a consumer that read before
      // its producer's completion would read the test's NaN poison
      if (tid == 0) {
        uint32_t x = jitter ^ (uint32_t)globaltimer() ^ ((uint32_t)blockIdx.x * 0x9e3779b9u) ^ ((uint32_t)tk * 0x85ebca6bu);
        x ^= x >> 15;
        x *= 0x2c1b3c6du;
        x ^= x >> 12;
        __nanosleep(x & 4095u);
      }
      __syncthreads();
    }
    unsigned long long t_start = 0;
    if (P.timing && tid == 0) t_start = globaltimer();
    if (S.b.w < 0) {
      // finaliser: product of rank-0 values, in double, member order
      if (tid == 0) {
        double re = 1.0, im = 0.0;
        for (int i = 0; i < S.b.n_mem; ++i) {
          const qtn_member_t m = P.members[S.b.mem_begin + i];
          QTN_CHECK(QTN_ARENA_OK(P, m.off), "finaliser member %d off %lld", i, (long long)m.off);
          const double2 v = (HI && m.off < n_hi) ? __ldg(Ahi + m.off) : widen(__ldcg(A + m.off));
          const double vr = v.x, vi = v.y;
          const double nr = re * vr - im * vi;
          const double ni = re * vi + im * vr;
          re = nr;
          im = ni;
        }
        P.results[2 * S.b.slot] = re;
        P.results[2 * S.b.slot + 1] = im;
      }
    } else {
      const int nm = S.b.n_mem;
      const int L = S.b.tile_bits;
      const int ns = 1 << S.b.k;
      const int nelem = 1 << L;
      if (tid < nm) S.base[tid] = S.off[tid] + (pext64((uint64_t)h, S.mhi[tid]) << S.pclo[tid]);
      __syncthreads();
      uint32_t hbits = 0;   // staged unrounded input members (bit i = member i)
      if (HI && n_hi)
        for (int i = 0; i < nm; ++i) hbits |= (uint32_t)S.hmode[i] << i;
      T* out = Aw + S.b.out_off + (uint64_t)h * (uint64_t)nelem;
      // threads cover (element, assignment) pairs, UJ per thread per round;
      // every member's loads of a round are issued before any multiply (one
      // L2 round trip per round instead of one per member)
      constexpr int UJ = 2;
      const int chunk = max(1, min(ns, SMALL_PROD_ELEMS / nelem));
      D acc = D{};
      for (int s0 = 0; s0 < ns; s0 += chunk) {
        const int cs = min(chunk, ns - s0);
        const int nu = cs * nelem;
        for (int u0 = tid; u0 < nu; u0 += UJ * NT) {
          int ue[UJ], us[UJ];
#pragma unroll
          for (int j = 0; j < UJ; ++j) {
            const int u = min(u0 + j * NT, nu - 1);
            ue[j] = u & (nelem - 1);
            us[j] = s0 + (u >> L);
          }
          // every member load of the round in flight together (input members
          // of complex64 programs: the narrowed copy, replaced at multiply
          // time by the unrounded value staged in shi / read from inputs_hi)
          T x[MAXM][UJ];
          int xe[MAXM][UJ];   // staged input member: element index into shi
#pragma unroll
          for (int i = 0; i < MAXM; ++i) {
            if (i < nm) {
#pragma unroll
              for (int j = 0; j < UJ; ++j) {
                const uint64_t o = S.base[i] + ((uint64_t)S.sig[i][us[j]] << S.pc[i]) +
                                   (S.pclo[i] == L ? (uint64_t)ue[j] : (uint64_t)pext32((uint32_t)ue[j], S.mlo[i]));
                QTN_CHECK(QTN_ARENA_OK(P, o), "small item %d member %d off %lld", cur, i, (long long)o);
                if (HI && ((hbits >> i) & 1u)) {
                  xe[i][j] = (int)(o - S.off[i]);
                } else {
                  x[i][j] = __ldcg(A + o);
                }
              }
            }
          }
#pragma unroll
          for (int j = 0; j < UJ; ++j) {
            D prod = D{};
#pragma unroll
            for (int i = 0; i < MAXM; ++i) {
              if (i < nm) {
                D xi;
                if (HI && ((hbits >> i) & 1u)) {
                  const int e = xe[i][j];
                  QTN_CHECK(e >= 0 && e < K2_HI_SLOT, "hi member %d index %d", i, e);
                  xi = shi[i * K2_HI_SLOT + e];
                } else {
                  xi = widen(x[i][j]);
                }
                prod = i == 0 ? xi : cmul(prod, xi);
              }
            }
            if (u0 + j * NT < nu) {
              QTN_CHECK((u0 + j * NT + 1) * (int)sizeof(D) <= (int)dyn_smem_bytes(), "sprod %d", u0 + j * NT);
              sprod[u0 + j * NT] = prod;
            }
          }
        }
        __syncthreads();
        if (tid < nelem)
          for (int c = 0; c < cs; ++c) acc = (s0 + c == 0) ? sprod[c * nelem + tid] : cadd(acc, sprod[c * nelem + tid]);
        __syncthreads();
      }
      QTN_CHECK(QTN_ARENA_OK(P, S.b.out_off + (uint64_t)h * nelem + nelem - 1), "small item %d out", cur);
      if (tid < nelem) narrow(acc, out[tid]);
    }
    __syncthreads();
    if (tid == 0) {
      ++pend_cnt;
      pend_item = cur;
      if (P.timing) {
        atomicMin(&P.timing[2 * cur], t_start);
        atomicMax(&P.timing[2 * cur + 1], globaltimer());
      }
      // the prefetched next ticket belongs to another item: publish now (a
      // dependent item may be waiting) instead of after the ticket search
      if (S.next >= S.item_end) {
        publish_tiles(&done[pend_item], pend_cnt);
        pend_cnt = 0;
      }
    }
  }
  // exit: publish, then the last block out zeroes the stage's counters
  if (tid == 0) {
    if (pend_cnt) {
      publish_tiles(&done[pend_item], pend_cnt);
    }
    // acq_rel: this block's publishes are ordered before its exit count, and
    // the last block out sees every block's publishes before it resets them
    unsigned v;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(v) : "l"(&ctl[1]) : "memory");
    S.last = (v == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (S.last) {
    __threadfence();
    for (int i = first + tid; i < first + count; i += NT) done[i] = 0u;
    if (tid == 0) {
      ctl[0] = 0u;
      ctl[1] = 0u;
    }
  }
}

// =========================================================================
// K1: large-item kernels
// =========================================================================
// A large item's descriptor and member records, passed to its K1 launch as
// a kernel parameter (known when the graph is built): the prologue needs no
// dependent global loads.
struct K1Item {
  qtn_bucket_t b;
  qtn_member_t mem[MAXM];
};

struct LargeCtx {
  qtn_bucket_t b;
  uint64_t off[MAXM];
  uint64_t mhi[MAXM];
  uint64_t base[MAXM];
  uint32_t mlo[MAXM];
  int32_t cls[MAXM];
  int32_t pc[MAXM];
  int32_t pclo[MAXM];
  int32_t nsig[MAXM];
  int32_t seglen[MAXM];
  int32_t seg[MAXM];       // smem element offset of the staged runs, -1 if not staged
  int32_t vlist[MAXM];     // varying members (compile-time count NV)
  int16_t sig[MAXM][MAXNS];
  int32_t gs[MAXM][MAXS];  // pext(est[st], mlo)
  int32_t gt[MAXM][NT];    // pext(eth[tid], mlo)
  int32_t eth[NT];         // tile offset of the thread's first result
  int32_t est[MAXS];       // tile offset of step st
  int32_t s0m;             // the streamed member (ST == 1)
  int32_t uoff;            // smem offset of U[s] (tile-uniform product)
  int32_t has_u;
  int32_t nbulk;
};

// Per-block preparation of a large item: member tables, smem layout, thread
// mapping (v -> bit 0 for c64, lane -> the next 5 bits for coalesced warp
// stores, warp and step bits -> the rest; step bits = the item's stmask).
template <typename R>
__device__ __forceinline__ void large_prep(LargeCtx& S, const qtn_program_t& P, int item, const K1Item& it,
                                           int nb0_expected) {
  using T = typename Cx<R>::T;
  constexpr int VEC = Cx<R>::VEC;
  constexpr int EPV = 16 / (int)sizeof(T);
  const int tid = threadIdx.x;
  if (tid == 0) S.b = it.b;   // published by the __syncthreads below
  const int nm = it.b.n_mem;
  const int L = it.b.tile_bits;
  const int k = it.b.k;
  if (tid < nm) {
    const qtn_member_t m = it.mem[tid];
    const uint32_t lowmask = (1u << L) - 1u;
    S.off[tid] = m.off;
    S.mlo[tid] = (uint32_t)(m.mask & lowmask);
    S.mhi[tid] = m.mask >> L;
    S.pc[tid] = __popcll(m.mask);
    S.pclo[tid] = __popc((uint32_t)(m.mask & lowmask));
    S.nsig[tid] = 1 << __popc(m.smask);
    S.seglen[tid] = 1 << S.pclo[tid];
    S.cls[tid] = (int)m.cls;
    for (int q = 0; q < (1 << k); ++q) S.sig[tid][q] = (int16_t)pext32((uint32_t)q, m.smask);
  }
  {
    constexpr int LB = (VEC == 2) ? 1 : 0;
    const uint32_t hi = ((1u << L) - 1u) & ~((1u << (LB + 5)) - 1u);
    uint32_t stm = it.b.stmask & hi;
    if (__popc(stm) != L - LB - 8) stm = hi & ~((1u << (LB + 8)) - 1u);
    const uint32_t wm = hi & ~stm;
    S.eth[tid] = (int)(((uint32_t)(tid & 31) << LB) | pdep32((uint32_t)(tid >> 5), wm));
    if (tid < MAXS) S.est[tid] = (int)pdep32((uint32_t)tid, stm);
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0, nv = 0, sm = -1, hu = 0, nb = 0;
    for (int i = 0; i < nm; ++i) {
      const int c = S.cls[i];
      if (c == QTN_CLS_STREAMED) {
        S.seg[i] = -1;
        if (sm < 0) sm = i;
      } else {
        S.seg[i] = acc;
        acc += S.nsig[i] * S.seglen[i];
        acc = (acc + EPV - 1) & ~(EPV - 1);   // 16-byte aligned runs (bulk copies)
        if (S.seglen[i] * (int)sizeof(T) >= 16) nb += S.nsig[i];
      }
      if (c == QTN_CLS_UNIFORM) hu = 1;
    }
    // varying members, those carrying result bit 0 first (their v pairs are
    // adjacent in smem: one 16-byte gather; c64 only)
    int nb0 = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i < nm; ++i)
        if (S.cls[i] == QTN_CLS_VARYING && (int)(S.mlo[i] & 1u) == 1 - pass) {
          S.vlist[nv++] = i;
          nb0 += 1 - pass;
        }
    // planner / kernel contract (always checked, once per block): the
    // specialisation must match the item's varying-member layout
    if (nb0_expected >= 0 && VEC == 2 && nb0 != nb0_expected) {
      printf("qtn_b200: item %d has %d bit-0 varying members, kernel variant expects %d\n", item, nb0, nb0_expected);
      __trap();
    }
    S.s0m = sm;
    S.has_u = hu;
    S.uoff = acc;
    S.nbulk = nb;
    QTN_CHECK((acc + MAXNS) * (int)sizeof(T) <= (int)dyn_smem_bytes(), "item %d staged %d elems > smem %u B", item,
              acc, dyn_smem_bytes());
    QTN_CHECK(nv <= MAXM && (L >= 32 ? false : true), "item %d bad layout", item);
    QTN_CHECK((1 << L) / (VEC * NT) <= MAXS, "item %d steps", item);
    QTN_CHECK(QTN_ARENA_OK(P, S.b.out_off + ((uint64_t)S.b.n_tiles << L) - 1), "item %d out range", item);
  }
  __syncthreads();
  if (tid < nm * MAXS) {
    const int i = tid / MAXS, st = tid % MAXS;
    S.gs[i][st] = (int)pext32((uint32_t)S.est[st], S.mlo[i]);
  }
  for (int i = 0; i < nm; ++i) S.gt[i][tid] = (int)pext32((uint32_t)S.eth[tid], S.mlo[i]);
  __syncthreads();
}

// Stage the non-streamed members of tile h: each run of >= 16 bytes is one
// bulk async copy completing on `bar`; shorter runs are plain loads.  Then
// U[s] = product of the tile-uniform members.
template <typename R>
__device__ __forceinline__ void large_stage(LargeCtx& S, const typename Cx<R>::T* A, typename Cx<R>::T* sseg,
                                            uint64_t* bar, uint32_t& phase, int h, const qtn_program_t& P_arena) {
  using T = typename Cx<R>::T;
  const int tid = threadIdx.x;
  const int nm = S.b.n_mem;
  const int ns = 1 << S.b.k;
  if (tid < nm) S.base[tid] = S.off[tid] + (pext64((uint64_t)h, S.mhi[tid]) << S.pclo[tid]);
  __syncthreads();
  if (tid == 0 && S.nbulk) {
    uint32_t bytes = 0;
    fence_proxy_async();   // order acquired generic-proxy data before async-proxy reads
    for (int i = 0; i < nm; ++i) {
      if (S.seg[i] < 0) continue;
      const uint32_t rb = (uint32_t)S.seglen[i] * (uint32_t)sizeof(T);
      if (rb < 16) continue;
      const T* src = A + S.base[i];
      for (int r = 0; r < S.nsig[i]; ++r) {
        QTN_CHECK(QTN_ARENA_OK(P_arena, S.base[i] + ((uint64_t)r << S.pc[i]) + S.seglen[i] - 1), "bulk src member %d run %d", i, r);
        QTN_CHECK(((uintptr_t)(src + ((uint64_t)r << S.pc[i])) & 15) == 0 && ((S.seg[i] + r * S.seglen[i]) * (int)sizeof(T)) % 16 == 0,
                  "bulk misaligned member %d run %d", i, r);
        bulk_g2s(sseg + S.seg[i] + r * S.seglen[i], src + ((uint64_t)r << S.pc[i]), rb, bar);
        bytes += rb;
      }
    }
    mbar_arrive_expect_tx(bar, bytes);
  }
  for (int i = 0; i < nm; ++i) {
    if (S.seg[i] < 0 || S.seglen[i] * (int)sizeof(T) >= 16) continue;
    const T* src = A + S.base[i];
    for (int q = tid; q < S.nsig[i]; q += NT) {
      QTN_CHECK(QTN_ARENA_OK(P_arena, S.base[i] + ((uint64_t)q << S.pc[i])), "short run member %d", i);
      sseg[S.seg[i] + q] = __ldcg(src + ((uint64_t)q << S.pc[i]));
    }
  }
  if (S.nbulk) {
    mbar_wait(bar, phase);
    phase ^= 1u;
  }
  __syncthreads();
  if (S.has_u && tid < ns) {
    T u = T{};
    bool first = true;
    for (int i = 0; i < nm; ++i) {
      if (S.cls[i] != QTN_CLS_UNIFORM) continue;
      const T x = sseg[S.seg[i] + S.sig[i][tid]];
      u = first ? x : cmul(u, x);
      first = false;
    }
    sseg[S.uoff + tid] = u;
  }
  __syncthreads();
}

// Compute tile h (after large_stage): fully unrolled over the NS summed
// assignments and the NV varying members; per-thread smem addresses and run
// offsets live in registers.
template <typename R, int NS, int NV, int ST, int NB0>
__device__ __forceinline__ void large_compute(const LargeCtx& S, const typename Cx<R>::T* __restrict__ A,
                                              const typename Cx<R>::T* sseg, typename Cx<R>::T* out) {
  using T = typename Cx<R>::T;
  using V = typename Cx<R>::V;
  constexpr int VEC = Cx<R>::VEC;
  const int tid = threadIdx.x;
  const int nm = S.b.n_mem;
  const int nst = (1 << S.b.tile_bits) / (VEC * NT);
  const T* qv[NV > 0 ? NV : 1];
  int ro[NV > 0 ? NV : 1][NS];
  int vi[NV > 0 ? NV : 1];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int i = S.vlist[j];
    vi[j] = i;
    qv[j] = sseg + S.seg[i] + S.gt[i][tid];
    QTN_CHECK(VEC == 1 || (int)(S.mlo[i] & 1u) == (j < NB0 ? 1 : 0), "vlist/NB0 mismatch item member %d", i);
#pragma unroll
    for (int c = 0; c < NS; ++c) ro[j][c] = S.sig[i][c] << S.pclo[i];
  }
  const T* sp = nullptr;
  int64_t sro[NS];
  if (ST) {
    const int sm = S.s0m;
    QTN_CHECK(sm >= 0, "ST variant without streamed member");
    sp = A + S.base[sm] + S.eth[tid];
#pragma unroll
    for (int c = 0; c < NS; ++c) sro[c] = (int64_t)S.sig[sm][c] << S.pc[sm];
  }
  // thread-invariant members (k <= 3): P[s] once per tile, with the
  // tile-uniform product U[s] folded in
  T P[NS][VEC];
  bool haveP = false;
  for (int i = 0; i < nm; ++i) {
    if (S.cls[i] != QTN_CLS_INVARIANT) continue;
    const T* q = sseg + S.seg[i] + S.gt[i][tid];
    const int bb = (int)(S.mlo[i] & 1u);
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      const T* qc = q + (S.sig[i][c] << S.pclo[i]);
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const T x = qc[v & bb];
        P[c][v] = haveP ? cmul(P[c][v], x) : x;
      }
    }
    haveP = true;
  }
  const bool hu0 = S.has_u;
  T U[NS];
#pragma unroll
  for (int c = 0; c < NS; ++c) U[c] = hu0 ? sseg[S.uoff + c] : T{};
  if (haveP && hu0) {
#pragma unroll
    for (int c = 0; c < NS; ++c)
#pragma unroll
      for (int v = 0; v < VEC; ++v) P[c][v] = cmul(U[c], P[c][v]);
  }
  const bool hu = hu0 && !haveP;
  // streamed loads of UNR steps are issued together before any of their
  // stores (the compiler cannot hoist them: loads and stores share the arena),
  // so each thread keeps UNR * NS 16-byte loads in flight
  constexpr int UNR = ST ? (NS <= 2 ? 4 : (NS == 4 ? 2 : 1)) : 1;
  for (int st0 = 0; st0 < nst; st0 += UNR) {
    T pre[UNR][NS][VEC];
    if (ST) {
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (st0 + u < nst) {
          const int est = S.est[st0 + u];
#pragma unroll
          for (int c = 0; c < NS; ++c) split(__ldcg(reinterpret_cast<const V*>(sp + est + sro[c])), pre[u][c]);
        }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int st = st0 + u;
      if (st >= nst) break;
      const int est = S.est[st];
      T prod[NS][VEC];
      bool started = false;
      if (ST) {
#pragma unroll
        for (int c = 0; c < NS; ++c)
#pragma unroll
          for (int v = 0; v < VEC; ++v) prod[c][v] = pre[u][c][v];
        started = true;
      }
      if (hu) {
#pragma unroll
        for (int c = 0; c < NS; ++c)
#pragma unroll
          for (int v = 0; v < VEC; ++v) prod[c][v] = started ? cmul(prod[c][v], U[c]) : U[c];
        started = true;
      }
      if (haveP) {
#pragma unroll
        for (int c = 0; c < NS; ++c)
#pragma unroll
          for (int v = 0; v < VEC; ++v) prod[c][v] = started ? cmul(prod[c][v], P[c][v]) : P[c][v];
        started = true;
      }
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const T* q = qv[j] + S.gs[vi[j]][st];
#pragma unroll
        for (int c = 0; c < NS; ++c) {
          QTN_CHECK((int)((q + ro[j][c]) - sseg) + VEC <= S.uoff + MAXNS &&
                        S.gt[vi[j]][tid] + S.gs[vi[j]][st] + ro[j][c] < S.nsig[vi[j]] * S.seglen[vi[j]],
                    "staged gather member %d", vi[j]);
          T x[VEC];
          if (VEC == 2 && j < NB0) {
            split(*reinterpret_cast<const V*>(q + ro[j][c]), x);   // adjacent v pair
          } else {
            x[0] = q[ro[j][c]];                                     // member constant in v
            x[VEC - 1] = x[0];
          }
#pragma unroll
          for (int v = 0; v < VEC; ++v) prod[c][v] = started ? cmul(prod[c][v], x[v]) : x[v];
        }
        started = true;
      }
      T acc[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        acc[v] = prod[0][v];
#pragma unroll
        for (int c = 1; c < NS; ++c) acc[v] = cadd(acc[v], prod[c][v]);
      }
      QTN_CHECK(S.eth[tid] + est + VEC <= (1 << S.b.tile_bits), "tile offset %d", S.eth[tid] + est);
      *reinterpret_cast<V*>(out + S.eth[tid] + est) = join(acc);
    }
  }
}

// Generic compute (any k, any member mix): summed assignments in chunks of 2,
// member parameters read from the block tables.
template <typename R>
__device__ __forceinline__ void large_compute_generic(const LargeCtx& S, const typename Cx<R>::T* __restrict__ A,
                                                      const typename Cx<R>::T* sseg, typename Cx<R>::T* out) {
  using T = typename Cx<R>::T;
  using V = typename Cx<R>::V;
  constexpr int VEC = Cx<R>::VEC;
  constexpr int SC = 2;
  const int tid = threadIdx.x;
  const int nm = S.b.n_mem;
  const int ns = 1 << S.b.k;
  const int nst = (1 << S.b.tile_bits) / (VEC * NT);
  for (int st = 0; st < nst; ++st) {
    const int e0 = S.eth[tid] + S.est[st];
    T acc[VEC];
    for (int s0 = 0; s0 < ns; s0 += SC) {
      T prod[SC][VEC];
      for (int i = 0; i < nm; ++i) {
        T x[SC][VEC];
        if (S.seg[i] < 0) {
          const T* q = A + S.base[i] + e0;
#pragma unroll
          for (int c = 0; c < SC; ++c)
            split(__ldcg(reinterpret_cast<const V*>(q + ((int64_t)S.sig[i][s0 + c] << S.pc[i]))), x[c]);
        } else {
          const T* q = sseg + S.seg[i] + S.gt[i][tid] + S.gs[i][st];
          const int bit0 = (int)(S.mlo[i] & 1u);
#pragma unroll
          for (int c = 0; c < SC; ++c) {
            const T* qc = q + (S.sig[i][s0 + c] << S.pclo[i]);
#pragma unroll
            for (int v = 0; v < VEC; ++v) x[c][v] = qc[v & bit0];
          }
        }
#pragma unroll
        for (int c = 0; c < SC; ++c)
#pragma unroll
          for (int v = 0; v < VEC; ++v) prod[c][v] = (i == 0) ? x[c][v] : cmul(prod[c][v], x[c][v]);
      }
#pragma unroll
      for (int c = 0; c < SC; ++c)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] = (s0 + c == 0) ? prod[c][v] : cadd(acc[v], prod[c][v]);
    }
    *reinterpret_cast<V*>(out + e0) = join(acc);
  }
}

// NS < 0: generic compute.
template <typename R, int NS, int NV, int ST, int NB0>
__device__ __forceinline__ void large_body(const qtn_program_t& P, int32_t item, const K1Item& it) {
  using T = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sseg = reinterpret_cast<T*>(smem_raw);
  __shared__ LargeCtx S;
  __shared__ uint64_t bar;
  const T* A = reinterpret_cast<const T*>(P.arena);
  T* Aw = reinterpret_cast<T*>(P.arena);
  const int tid = threadIdx.x;
  pdl_launch_dependents();
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  large_prep<R>(S, P, item, it, NS > 0 ? NB0 : -1);   // static tables only
  pdl_wait();                  // predecessors complete: their outputs are readable
  unsigned long long t_start = 0;
  if (P.timing && tid == 0) t_start = globaltimer();
  uint32_t phase = 0;
  const int ntiles = S.b.n_tiles;
  const uint64_t nelem = 1ull << S.b.tile_bits;
  for (int h = blockIdx.x; h < ntiles; h += gridDim.x) {
    large_stage<R>(S, A, sseg, &bar, phase, h, P);
    T* out = Aw + S.b.out_off + (uint64_t)h * nelem;
    if (NS > 0)
      large_compute<R, (NS > 0 ? NS : 2), NV, ST, NB0>(S, A, sseg, out);
    else
      large_compute_generic<R>(S, A, sseg, out);
    __syncthreads();
  }
  if (P.timing && tid == 0) {
    atomicMin(&P.timing[2 * item], t_start);
    atomicMax(&P.timing[2 * item + 1], globaltimer());
  }
}

// One kernel per element type so each gets its own register budget: complex64
// runs best with the compiler's default allocation, complex128 with a cap
// that keeps 3 blocks resident (measured on cfg-2: 0.671 -> 0.605 ms).
#ifdef K1_C64_MINB
#define K1_C64_BOUNDS __launch_bounds__(NT, K1_C64_MINB)
#else
#define K1_C64_BOUNDS __launch_bounds__(NT)
#endif
template <int NS, int NV, int ST, int NB0>
__global__ void K1_C64_BOUNDS large_kernel_c64(const qtn_program_t P, int32_t item, const __grid_constant__ K1Item it) {
  large_body<float, NS, NV, ST, NB0>(P, item, it);
}
template <int NS, int NV, int ST, int NB0>
__global__ void __launch_bounds__(NT, 3) large_kernel_c128(const qtn_program_t P, int32_t item,
                                                           const __grid_constant__ K1Item it) {
  large_body<double, NS, NV, ST, NB0>(P, item, it);
}
template <typename R, int NS, int NV, int ST, int NB0>
struct LargeK {
  static constexpr auto fn = large_kernel_c64<NS, NV, ST, NB0>;
};
template <int NS, int NV, int ST, int NB0>
struct LargeK<double, NS, NV, ST, NB0> {
  static constexpr auto fn = large_kernel_c128<NS, NV, ST, NB0>;
};

// ---- input gather: raw tensors (pinned host, mapped) -> canonical image ----
template <typename R>
__global__ void __launch_bounds__(NT) gather_kernel(const double2* __restrict__ raw, const int64_t* __restrict__ src,
                                                   const int64_t* __restrict__ dst, int64_t n,
                                                   typename Cx<R>::T* __restrict__ arena, double2* __restrict__ hi) {
  pdl_launch_dependents();
  for (int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x; t < n; t += (int64_t)gridDim.x * NT) {
    const double2 v = raw[src[t]];
    const int64_t o = dst[t];
    narrow(v, arena[o]);
    if (hi) hi[o] = v;
  }
}

// ---- permutation (tensors entering a program in a non-canonical layout) ----
struct PermStrides {
  int64_t s[QTN_MAX_WIDTH + 4];
};

template <typename RS, typename RD>
__global__ void permute_kernel(const typename Cx<RS>::T* __restrict__ src, int64_t src_off,
                               typename Cx<RD>::T* __restrict__ dst, int rank, PermStrides st, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    int64_t o = src_off;
    for (int j = 0; j < rank; ++j) o += (int64_t)((e >> j) & 1ull) * st.s[j];
    const typename Cx<RS>::T v = src[o];
    typename Cx<RD>::T w;
    w.x = (RD)v.x;
    w.y = (RD)v.y;
    dst[e] = w;
  }
}

// =========================================================================
// host side: kernel selection, launch configuration, graphs
// =========================================================================
using LargeFn = void (*)(const qtn_program_t, int32_t, K1Item);

template <typename R, int NS, int NV, int ST>
LargeFn large_fn_nb0(int nb0) {
  if (Cx<R>::VEC == 1) return LargeK<R, NS, NV, ST, 0>::fn;
  switch (nb0) {
    case 0: return LargeK<R, NS, NV, ST, 0>::fn;
    case 1: return NV >= 1 ? LargeK<R, NS, NV, ST, (NV >= 1 ? 1 : 0)>::fn : nullptr;
    case 2: return NV >= 2 ? LargeK<R, NS, NV, ST, (NV >= 2 ? 2 : 0)>::fn : nullptr;
    case 3: return NV >= 3 ? LargeK<R, NS, NV, ST, (NV >= 3 ? 3 : 0)>::fn : nullptr;
    case 4: return NV >= 4 ? LargeK<R, NS, NV, ST, (NV >= 4 ? 4 : 0)>::fn : nullptr;
    default: return nullptr;
  }
}

template <typename R, int NS, int ST>
LargeFn large_fn_nv(int nv, int nb0) {
  switch (nv) {
    case 0: return large_fn_nb0<R, NS, 0, ST>(nb0);
    case 1: return large_fn_nb0<R, NS, 1, ST>(nb0);
    case 2: return large_fn_nb0<R, NS, 2, ST>(nb0);
    case 3: return large_fn_nb0<R, NS, 3, ST>(nb0);
    case 4: return large_fn_nb0<R, NS, 4, ST>(nb0);
    default: return nullptr;
  }
}

// variant = log2(2^k) | nv << 4 | streamed << 8 | nb0 << 12 (see qtn_b200.h)
template <typename R>
LargeFn large_fn(int variant) {
  LargeFn f = nullptr;
  if (variant >= 0) {
    const int ks = variant & 15, nv = (variant >> 4) & 15, st = (variant >> 8) & 1, nb0 = (variant >> 12) & 15;
    if (ks == 1) f = st ? large_fn_nv<R, 2, 1>(nv, nb0) : large_fn_nv<R, 2, 0>(nv, nb0);
    else if (ks == 2) f = st ? large_fn_nv<R, 4, 1>(nv, nb0) : large_fn_nv<R, 4, 0>(nv, nb0);
    else if (ks == 3) f = st ? large_fn_nv<R, 8, 1>(nv, nb0) : large_fn_nv<R, 8, 0>(nv, nb0);
  }
  return f ? f : LargeK<R, -1, 0, 0, 0>::fn;
}

int sm_count() {
  int dev = 0, nsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return nsm;
}

int resident_grid(const void* fn, int smem, int* grid) {
  // the attribute only ever grows: other nodes of the same kernel may need more
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return cuda_err(e, "cudaFuncGetAttributes");
  if (smem > fa.maxDynamicSharedSizeBytes) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_err(e, "cudaFuncSetAttribute");
  }
  int nb = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, NT, smem);
  if (e != cudaSuccess) return cuda_err(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  if (nb < 1) return set_err(QTN_E_UNSUPPORTED, "kernel cannot be resident with %d B smem", smem);
  *grid = nb * sm_count();
  return QTN_OK;
}

struct LaunchSpec {
  const void* fn;
  int grid;
  int smem;
  void* args[6];
  // storage for the arguments (the graph copies them at node creation)
  qtn_program_t prog;
  int32_t a0, a1, a2;
  uint32_t a3;
  uint32_t* ctl;
  K1Item k1item;                       // K1 node: its item (kernel parameter)
  std::vector<unsigned char> k3plan;   // K3 node: its Plan (kernel parameter)
};

int check_program(const qtn_program_t* p) {
  if (!p) return set_err(QTN_E_INVALID, "null program");
  if (p->dtype != QTN_C64 && p->dtype != QTN_C128) return set_err(QTN_E_INVALID, "bad dtype %d", p->dtype);
  if (p->n_buckets < 0 || p->n_nodes < 0) return set_err(QTN_E_INVALID, "negative sizes");
  if (p->n_buckets > 0 && (!p->buckets || !p->tick_begin || !p->ctrl))
    return set_err(QTN_E_INVALID, "null device table");
  return QTN_OK;
}

// Fill the launch of node `ni` (itm: host copy of a LARGE node's item + members).
int make_launch(const qtn_program_t* p, const qtn_node_t* nd, int ni, const K1Item* itm, LaunchSpec* L) {
  L->prog = *p;
  L->smem = nd->smem_bytes;
  if (L->smem < 0 || L->smem > 227 * 1024) return set_err(QTN_E_INVALID, "node smem %d", L->smem);
  int rc;
  if (nd->kind == QTN_NODE_SMALL) {
    L->fn = p->dtype == QTN_C64 ? (const void*)small_kernel<float> : (const void*)small_kernel<double>;
    rc = resident_grid(L->fn, L->smem, &L->grid);
    if (rc) return rc;
    if (nd->n_tickets < L->grid) L->grid = nd->n_tickets > 0 ? nd->n_tickets : 1;
    // prog->grid > 0 caps the stage's persistent grid (schedule-independence
    // tests: any number of blocks must give the same bits)
    if (p->grid > 0 && p->grid < L->grid) L->grid = p->grid;
    L->a0 = nd->first;
    L->a1 = nd->count;
    L->a2 = nd->n_tickets;
    L->ctl = p->ctrl + 2 * ni;
    L->a3 = (uint32_t)qtn_knobs().k2_jitter;
    L->args[0] = &L->prog;
    L->args[1] = &L->a0;
    L->args[2] = &L->a1;
    L->args[3] = &L->a2;
    L->args[4] = &L->ctl;
    L->args[5] = &L->a3;
  } else if (nd->kind == QTN_NODE_LARGE) {
    L->fn = p->dtype == QTN_C64 ? (const void*)large_fn<float>(nd->variant)
                                : (const void*)large_fn<double>(nd->variant);
    rc = resident_grid(L->fn, L->smem, &L->grid);
    if (rc) return rc;
    if (!itm) return set_err(QTN_E_INVALID, "large node without item");
    const int32_t n_tiles = itm->b.n_tiles;
    if (n_tiles < L->grid) L->grid = n_tiles > 0 ? n_tiles : 1;
    L->a0 = nd->first;
    L->k1item = *itm;
    L->args[0] = &L->prog;
    L->args[1] = &L->a0;
    L->args[2] = &L->k1item;
  } else {
    return set_err(QTN_E_INVALID, "bad node kind %d", nd->kind);
  }
  return QTN_OK;
}

}  // namespace

int qtn_internal_set_error(int code, const char* msg) { return set_err(code, "%s", msg); }

// K3 (bucket_strided.cu) as a program node: expansion items whose staged
// members K1 would gather per tile
size_t qtn_k3_plan_bytes();
size_t qtn_k4_plan_bytes();
size_t qtn_k5_plan_bytes();
int qtn_k5_node(const qtn_bucket_desc_t* d, int max_e, unsigned long long* timing, int32_t item, void* plan,
                const void** fn, int* grid, int* smem);
int qtn_k4_node(const qtn_bucket_desc_t* d, int min_e, unsigned long long* timing, int32_t item, void* plan,
                const void** fn, int* grid, int* smem);
int qtn_k3_node(const qtn_bucket_desc_t* d, unsigned long long* timing, int32_t item, void* plan, const void** fn,
                int* grid, int* smem);
size_t qtn_k6_plan_bytes();
int qtn_k6_node(const qtn_bucket_desc_t* dp, const qtn_bucket_desc_t* dc, int ipc, unsigned long long* timing,
                int32_t item_p, int32_t item_c, void* plan, const void** fn, int* grid, int* smem);

namespace {

// one knob: the environment value if it parses as an integer in [lo, hi],
// else the default (a rejected value is reported once on stderr)
int knob(const char* name, int dflt, int lo, int hi) {
  const char* v = getenv(name);
  if (!v || !v[0]) return dflt;
  char* end = nullptr;
  const long x = strtol(v, &end, 10);
  if (*end != '\0' || x < lo || x > hi) {
    fprintf(stderr, "qtn_b200: ignoring %s=%s (integer in [%d, %d] expected); using %d\n", name, v, lo, hi, dflt);
    return dflt;
  }
  return (int)x;
}

QtnKnobs read_knobs() {
  QtnKnobs k;
  k.k3_route = knob("QTN_K3_ROUTE", -1, -1, 64);
  k.k4_min_e = knob("QTN_K4", 1, 0, 4);
  k.k4_all = knob("QTN_K4_ALL", -1, -1, 1);
  k.k5 = knob("QTN_K5", 1, 0, 2);
  k.pdl = knob("QTN_PDL", 1, 0, 1);
  k.k3_tcap = knob("QTN_K3_TCAP", 0, 0, 16);
  k.k3_stage_kb = knob("QTN_K3_STAGE_KB", 40, 8, 200);
  k.k3_run = knob("QTN_K3_RUN", 128, 16, 4096);
  k.k3_v1 = knob("QTN_K3_V1", 0, 0, 1);
  k.k3_ulim = knob("QTN_K3_ULIM", 5, 0, 8);
  k.k3_inv2 = knob("QTN_K3_INV2", 1, 0, 1);
  k.k6_min_w = knob("QTN_K6", 18, 0, 40);
  k.k2_jitter = knob("QTN_K2_JITTER", 0, 0, 1 << 30);
  return k;
}


// Route a large item to K3?  QTN_K3_ROUTE: 0 never, 1 merged expansion items
// (k >= 2, >= 2 varying staged members), 2 every large item, >= 10: every
// large item at least that wide.  Default (measured on B200):
// complex64 keeps K1 (K3 on merged expansions: cfg-2 -0.3 %, 45-cone graph
// +2 %, cfg-3 +4 %); complex128 routes items of width >= 20 to K3 (cfg-2
// 0.593 -> 0.497 ms, 45-cone graph +0.8 %).
bool k3_route(const qtn_bucket_t& b, const qtn_member_t* mem, int dtype) {
  const int env = qtn_knobs().k3_route;
  const int mode = env >= 0 ? env : (dtype == QTN_C64 ? 0 : 20);
  if (mode == 0 || b.w < 0 || b.k > 3 || b.w > 31 || b.n_mem > QTN_MAX_MEMBERS) return false;
  if (mode == 2) return true;
  if (mode >= 10) return b.w >= mode;   // A/B: every large item at least that wide
  int nv = 0;
  for (int i = 0; i < b.n_mem; ++i) nv += mem[b.mem_begin + i].cls == QTN_CLS_VARYING;
  return b.k >= 2 && nv >= 2;
}

// canonical layout -> K3 strides: member offset (pext(s, smask) << popc(mask)) + pext(r, mask)
void k3_desc(const qtn_program_t* p, const qtn_bucket_t& b, const qtn_member_t* mem, qtn_bucket_desc_t* d) {
  const size_t esz = p->dtype == QTN_C64 ? 8 : 16;
  memset(d, 0, sizeof(*d));
  d->dtype = p->dtype;
  d->w = b.w;
  d->k = b.k;
  d->n_mem = b.n_mem;
  d->out = (char*)p->arena + b.out_off * esz;
  for (int i = 0; i < b.n_mem; ++i) {
    const qtn_member_t& m = mem[b.mem_begin + i];
    d->mem[i].data = (const char*)p->arena + m.off * esz;
    const int pc = __builtin_popcountll(m.mask);
    int r = 0;
    for (int bit = 0; bit < b.w; ++bit)
      if ((m.mask >> bit) & 1) d->mem[i].strides[bit] = (int64_t)1 << r++;
    int q = 0;
    for (int j = 0; j < b.k; ++j)
      if ((m.smask >> j) & 1) d->mem[i].strides[b.w + j] = (int64_t)1 << (pc + q++);
  }
}

}  // namespace

const QtnKnobs& qtn_knobs() {
  static const QtnKnobs k = read_knobs();   // thread-safe one-time init
  return k;
}

struct qtn_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int32_t kinds[6] = {0, 0, 0, 0, 0, 0};   // kernels K1, K2, K3, K4, K5, K6 in the graph
  std::vector<int32_t> node_kind;          // per node: 0 K1, 1 K2, 2 K3, 3 K4, 4 K5, 5 K6
};

extern "C" {

int qtn_abi_version(void) { return QTN_ABI_VERSION; }

const char* qtn_route_config(void) {
  static const std::string txt = [] {
    const QtnKnobs& k = qtn_knobs();
    char buf[512];
    snprintf(buf, sizeof(buf),
             "k3_route=%d k4_min_e=%d k4_all=%d k5=%d pdl=%d k3_tcap=%d k3_stage_kb=%d k3_run=%d k3_v1=%d k3_ulim=%d "
             "k3_inv2=%d k6_min_w=%d k2_jitter=%d",
             k.k3_route, k.k4_min_e, k.k4_all, k.k5, k.pdl, k.k3_tcap, k.k3_stage_kb, k.k3_run, k.k3_v1, k.k3_ulim,
             k.k3_inv2, k.k6_min_w, k.k2_jitter);
    return std::string(buf);
  }();
  return txt.c_str();
}

const char* qtn_last_error(void) { return g_err.c_str(); }

int qtn_device_count(int* count) {
  if (!count) return set_err(QTN_E_INVALID, "null count");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *count = n;
  return QTN_OK;
}

int qtn_program_reset(const qtn_program_t* p, void* stream) {
  int rc = check_program(p);
  if (rc) return rc;
  const size_t words = 2 * (size_t)p->n_nodes + (size_t)p->n_buckets;
  const cudaError_t e = cudaMemsetAsync(p->ctrl, 0, sizeof(uint32_t) * words, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_err(e, "cudaMemsetAsync(ctrl)");
  return QTN_OK;
}

int qtn_node_launch(const qtn_program_t* p, const qtn_node_t* nd, int32_t ni, void* stream) {
  int rc = check_program(p);
  if (rc) return rc;
  if (!nd) return set_err(QTN_E_INVALID, "null node");
  if (nd->kind == QTN_NODE_LARGE && nd->count == 2) {
    // producer / consumer pair: the two items in order (K1 each)
    qtn_node_t sub[2] = {*nd, *nd};
    sub[0].count = sub[1].count = 1;
    sub[1].first = nd->first + 1;
    sub[0].variant = nd->n_tickets;
    sub[0].n_tickets = sub[1].n_tickets = 0;
    qtn_bucket_t bp;
    if (nd->first < 0 || nd->first + 1 >= p->n_buckets) return set_err(QTN_E_INVALID, "item %d out of range", nd->first);
    const cudaError_t e = cudaMemcpy(&bp, p->buckets + nd->first, sizeof(bp), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_err(e, "cudaMemcpy(item)");
    sub[0].smem_bytes = (int32_t)((bp.smem_elems * (p->dtype == QTN_C64 ? 8 : 16) + 15) / 16 * 16);
    for (int j = 0; j < 2; ++j) {
      rc = qtn_node_launch(p, &sub[j], ni, stream);
      if (rc) return rc;
    }
    return QTN_OK;
  }
  K1Item itm{};
  if (nd->kind == QTN_NODE_LARGE) {
    if (nd->count != 1) return set_err(QTN_E_INVALID, "large node with %d items", nd->count);
    if (nd->first < 0 || nd->first >= p->n_buckets) return set_err(QTN_E_INVALID, "item %d out of range", nd->first);
    cudaError_t e = cudaMemcpy(&itm.b, p->buckets + nd->first, sizeof(itm.b), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_err(e, "cudaMemcpy(item)");
    if (itm.b.n_mem < 0 || itm.b.n_mem > MAXM) return set_err(QTN_E_INVALID, "item %d: %d members", nd->first, itm.b.n_mem);
    if (itm.b.n_mem > 0) {
      e = cudaMemcpy(itm.mem, p->members + itm.b.mem_begin, sizeof(qtn_member_t) * itm.b.n_mem, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_err(e, "cudaMemcpy(members)");
    }
  }
  LaunchSpec L;
  rc = make_launch(p, nd, ni, nd->kind == QTN_NODE_LARGE ? &itm : nullptr, &L);
  if (rc) return rc;
  const cudaError_t e = cudaLaunchKernel(L.fn, dim3(L.grid), dim3(NT), L.args, L.smem, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_err(e, "cudaLaunchKernel");
  return QTN_OK;
}

int qtn_graph_create(const qtn_program_t* p, const qtn_node_t* nodes, int32_t n_nodes, const int32_t* node_deps,
                     qtn_graph_t** out) {
  return qtn_graph_create_io(p, nodes, n_nodes, node_deps, nullptr, out);
}

int qtn_graph_create_io(const qtn_program_t* p, const qtn_node_t* nodes, int32_t n_nodes, const int32_t* node_deps,
                        const qtn_graph_io_t* io, qtn_graph_t** out) {
  int rc = check_program(p);
  if (rc) return rc;
  std::vector<qtn_bucket_t> items(p->n_buckets);
  if (p->n_buckets) {
    const cudaError_t e =
        cudaMemcpy(items.data(), p->buckets, sizeof(qtn_bucket_t) * items.size(), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_err(e, "cudaMemcpy(items)");
  }
  int64_t n_members = 0;
  for (const qtn_bucket_t& b : items) n_members = std::max<int64_t>(n_members, (int64_t)b.mem_begin + std::max(0, b.n_mem));
  std::vector<qtn_member_t> mems(n_members);
  if (n_members && p->members) {
    const cudaError_t e = cudaMemcpy(mems.data(), p->members, sizeof(qtn_member_t) * mems.size(), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_err(e, "cudaMemcpy(members)");
  }
  return qtn_graph_create_host(p, items.data(), mems.data(), n_members, nodes, n_nodes, node_deps, io, out);
}

int qtn_graph_create_host(const qtn_program_t* p, const qtn_bucket_t* items, const qtn_member_t* mems_in,
                          int64_t n_host_members, const qtn_node_t* nodes, int32_t n_nodes, const int32_t* node_deps,
                          const qtn_graph_io_t* io, qtn_graph_t** out) {
  int rc = check_program(p);
  if (rc) return rc;
  if (!out || (n_nodes > 0 && !nodes) || (p->n_buckets > 0 && !items)) return set_err(QTN_E_INVALID, "null argument");
  for (int32_t i = 0; i < p->n_buckets; ++i) {
    const qtn_bucket_t& b = items[i];
    if (b.n_mem < 0 || b.mem_begin < 0 || (int64_t)b.mem_begin + b.n_mem > n_host_members || (b.n_mem > 0 && !mems_in))
      return set_err(QTN_E_INVALID, "item %d: members [%d, +%d) outside the %lld host members", i, b.mem_begin,
                     b.n_mem, (long long)n_host_members);
  }
  // the K3 route wants a member array it can index (empty when there is none)
  const qtn_member_t* mems_ptr = mems_in;
  const bool have_mems = n_host_members > 0 && mems_in;
  qtn_graph* g = new qtn_graph();
  cudaError_t e = cudaGraphCreate(&g->graph, 0);
  if (e != cudaSuccess) {
    delete g;
    return cuda_err(e, "cudaGraphCreate");
  }
  std::vector<cudaGraphNode_t> gn(n_nodes);
  std::vector<LaunchSpec> specs(n_nodes);
  // optional input upload: every kernel node without a predecessor waits for it
  cudaGraphNode_t h2d = nullptr;
  bool h2d_kernel = false;   // h2d is the device gather kernel (a PDL edge can follow it)
  if (io && io->n_gather > 0) {
    // device-side gather of the raw inputs (mapped pinned host memory)
    if (!io->gather_raw || !io->gather_src || !io->gather_dst || !p->arena) {
      qtn_graph_destroy(g);
      return set_err(QTN_E_INVALID, "gather: null pointer");
    }
    static thread_local struct {
      const void* raw;
      const int64_t* src;
      const int64_t* dst;
      int64_t n;
      void* arena;
      void* hi;
    } ga;
    ga = {io->gather_raw, io->gather_src, io->gather_dst, io->n_gather, p->arena, const_cast<void*>(p->inputs_hi)};
    void* args[] = {&ga.raw, &ga.src, &ga.dst, &ga.n, &ga.arena, &ga.hi};
    cudaKernelNodeParams kp = {};
    kp.func = p->dtype == QTN_C64 ? (void*)gather_kernel<float> : (void*)gather_kernel<double>;
    const int64_t blocks = std::min<int64_t>((io->n_gather + NT - 1) / NT, (int64_t)sm_count() * 4);
    kp.gridDim = dim3((unsigned)std::max<int64_t>(1, blocks));
    kp.blockDim = dim3(NT);
    kp.sharedMemBytes = 0;
    kp.kernelParams = args;
    e = cudaGraphAddKernelNode(&h2d, g->graph, nullptr, 0, &kp);   // parameters copied at node creation
    h2d_kernel = true;
    if (e != cudaSuccess) {
      qtn_graph_destroy(g);
      return cuda_err(e, "cudaGraphAddKernelNode(gather)");
    }
  } else if (io && io->h2d_bytes > 0) {
    e = cudaGraphAddMemcpyNode1D(&h2d, g->graph, nullptr, 0, io->h2d_dst, io->h2d_src, (size_t)io->h2d_bytes,
                                 cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      qtn_graph_destroy(g);
      return cuda_err(e, "cudaGraphAddMemcpyNode1D(h2d)");
    }
  }
  const QtnKnobs& route = qtn_knobs();
  const bool use_pdl = route.pdl != 0;
  const size_t esz = p->dtype == QTN_C64 ? 8 : 16;
  // Launch of one item-level node `sub` (a SMALL stage, or ONE large item):
  // K2 / K1 from make_launch, then the K5 / K4 / K3 routes for large items.
  // fam: 0 K1, 1 K2, 2 K3, 3 K4, 4 K5.
  auto route_node = [&](const qtn_node_t& sub, int ni, LaunchSpec& spec, int& fam) -> int {
    K1Item itm{};
    if (sub.kind == QTN_NODE_LARGE) {
      itm.b = items[sub.first];
      if (itm.b.n_mem < 0 || itm.b.n_mem > MAXM) return set_err(QTN_E_INVALID, "node %d: item with %d members", ni, itm.b.n_mem);
      for (int j = 0; j < itm.b.n_mem; ++j) itm.mem[j] = mems_ptr[itm.b.mem_begin + j];
    }
    int rc2 = make_launch(p, &sub, ni, sub.kind == QTN_NODE_LARGE ? &itm : nullptr, &spec);
    if (rc2) return rc2;
    fam = sub.kind == QTN_NODE_LARGE ? 0 : 1;
    if (sub.kind != QTN_NODE_LARGE || !p->arena || !have_mems) return QTN_OK;
    const qtn_bucket_t& it = items[sub.first];
    auto take = [&](std::vector<unsigned char>&& plan, const void* fn, int grid, int smem, int f) {
      spec.k3plan = std::move(plan);
      spec.fn = fn;
      spec.grid = grid;
      spec.smem = smem;
      spec.args[0] = spec.k3plan.data();
      fam = f;
    };
    qtn_bucket_desc_t d;
    k3_desc(p, it, mems_ptr, &d);
    const void* fn = nullptr;
    int grid = 0, smem = 0;
    // K5: streaming items (one member carries every result bit)
    if (route.k5 && it.k >= 1) {
      std::vector<unsigned char> plan(qtn_k5_plan_bytes());
      if (qtn_k5_node(&d, route.k5 >= 2 ? 4 : 0, p->timing, sub.first, plan.data(), &fn, &grid, &smem) == QTN_OK) {
        take(std::move(plan), fn, grid, smem, 4);
        return QTN_OK;
      }
    }
    // K4: expansion items of one dominant member (QTN_K4 = fewest expansion
    // bits routed, 0 = never); non-expansion items too: complex128 by default
    // (cfg-2 0.3575 -> 0.3519 ms), not complex64 (its streaming items stay
    // faster in K1); QTN_K4_ALL overrides
    if (route.k4_min_e > 0 && it.k >= 1 && it.w >= 12) {
      std::vector<unsigned char> plan(qtn_k4_plan_bytes());
      const bool k4_all = route.k4_all >= 0 ? route.k4_all != 0 : p->dtype == QTN_C128;
      if (qtn_k4_node(&d, k4_all ? 0 : route.k4_min_e, p->timing, sub.first, plan.data(), &fn, &grid, &smem) ==
          QTN_OK) {
        take(std::move(plan), fn, grid, smem, 3);
        return QTN_OK;
      }
    }
    if (k3_route(it, mems_ptr, p->dtype)) {
      std::vector<unsigned char> plan(qtn_k3_plan_bytes());
      if (qtn_k3_node(&d, p->timing, sub.first, plan.data(), &fn, &grid, &smem) == QTN_OK)
        take(std::move(plan), fn, grid, smem, 2);
      // else: K1 stays (the K3 planner declined this item)
    }
    return QTN_OK;
  };
  auto add_kernel = [&](const LaunchSpec& spec, const std::vector<cudaGraphNode_t>& deps, bool first_node,
                        cudaGraphNode_t* node) -> int {
    cudaKernelNodeParams kp = {};
    kp.func = const_cast<void*>(spec.fn);
    kp.gridDim = dim3(spec.grid);
    kp.blockDim = dim3(NT);
    kp.sharedMemBytes = spec.smem;
    kp.kernelParams = const_cast<void**>(spec.args);
    // a K2 stage after the device gather follows it over a programmatic edge
    // (its ticket, records and L2 warm-up overlap the gather's PCIe reads; it
    // reads no input before griddepcontrol.wait); other kernels may read
    // input members in their prologue, so they wait for the gather's end
    const bool k2 = spec.fn == (const void*)small_kernel<float> || spec.fn == (const void*)small_kernel<double>;
    const bool pdl_in = h2d && first_node && h2d_kernel && use_pdl && k2;
    cudaError_t e2 = cudaGraphAddKernelNode(node, g->graph, (h2d && first_node && !pdl_in) ? &h2d : nullptr,
                                            (h2d && first_node && !pdl_in) ? 1 : 0, &kp);
    if (e2 != cudaSuccess) return cuda_err(e2, "cudaGraphAddKernelNode");
    if (pdl_in) {
      cudaGraphEdgeData ed = {};
      ed.from_port = cudaGraphKernelNodePortProgrammatic;
      ed.type = cudaGraphDependencyTypeProgrammatic;
      e2 = cudaGraphAddDependencies_v2(g->graph, &h2d, node, &ed, 1);
      if (e2 != cudaSuccess) return cuda_err(e2, "cudaGraphAddDependencies_v2(gather)");
    }
    // programmatic edges (PDL): the kernels call griddepcontrol.wait before
    // reading predecessor outputs
    for (cudaGraphNode_t from : deps) {
      cudaGraphEdgeData ed = {};
      ed.from_port = use_pdl ? cudaGraphKernelNodePortProgrammatic : cudaGraphKernelNodePortDefault;
      ed.type = use_pdl ? cudaGraphDependencyTypeProgrammatic : cudaGraphDependencyTypeDefault;
      e2 = cudaGraphAddDependencies_v2(g->graph, &from, node, &ed, 1);
      if (e2 != cudaSuccess) return cuda_err(e2, "cudaGraphAddDependencies_v2");
    }
    return QTN_OK;
  };
  for (int i = 0; i < n_nodes; ++i) {
    const qtn_node_t& nd = nodes[i];
    const bool pair = nd.kind == QTN_NODE_LARGE && nd.count == 2;
    if (nd.kind == QTN_NODE_LARGE &&
        (nd.first < 0 || nd.first + (pair ? 1 : 0) >= p->n_buckets || (nd.count != 1 && nd.count != 2))) {
      qtn_graph_destroy(g);
      return set_err(QTN_E_INVALID, "node %d: items [%d, +%d) out of range", i, nd.first, nd.count);
    }
    std::vector<cudaGraphNode_t> deps;
    for (int d = 0; d < nd.n_dep; ++d) {
      const int j = node_deps[nd.dep_begin + d];
      if (j < 0 || j >= i) {
        qtn_graph_destroy(g);
        return set_err(QTN_E_INVALID, "node %d: dependency %d is not an earlier node", i, j);
      }
      deps.push_back(gn[j]);
    }
    int fam = 0;
    if (pair) {
      // producer / consumer pair (the producer's result is read by the
      // consumer only): K6 keeps the producer's result out of HBM; otherwise
      // the two items run as two kernels in sequence
      const qtn_bucket_t& bp = items[nd.first];
      const qtn_bucket_t& bc = items[nd.first + 1];
      bool fused = false;
      if (route.k6_min_w > 0 && bp.w >= route.k6_min_w && p->arena && have_mems) {
        int ipc = -1;
        for (int j = 0; j < bc.n_mem; ++j)
          if (mems_ptr[bc.mem_begin + j].off == bp.out_off) ipc = j;
        qtn_bucket_desc_t dp, dc;
        k3_desc(p, bp, mems_ptr, &dp);
        k3_desc(p, bc, mems_ptr, &dc);
        std::vector<unsigned char> plan(qtn_k6_plan_bytes());
        const void* fn = nullptr;
        int grid = 0, smem = 0;
        if (ipc >= 0 && qtn_k6_node(&dp, &dc, ipc, p->timing, nd.first, nd.first + 1, plan.data(), &fn, &grid,
                                    &smem) == QTN_OK) {
          specs[i].prog = *p;
          specs[i].k3plan = std::move(plan);
          specs[i].fn = fn;
          specs[i].grid = grid;
          specs[i].smem = smem;
          specs[i].args[0] = specs[i].k3plan.data();
          fam = 5;
          fused = true;
          rc = add_kernel(specs[i], deps, nd.n_dep == 0, &gn[i]);
        }
      }
      if (!fused) {
        qtn_node_t sp = nd, sc = nd;
        sp.count = sc.count = 1;
        sc.first = nd.first + 1;
        sp.variant = nd.n_tickets;   // LARGE pairs carry the producer's K1 variant here
        sp.n_tickets = sc.n_tickets = 0;
        sp.smem_bytes = (int32_t)((bp.smem_elems * esz + 15) / 16 * 16);
        LaunchSpec lp;
        int fp = 0;
        cudaGraphNode_t np_ = nullptr;
        rc = route_node(sp, i, lp, fp);
        if (!rc) rc = add_kernel(lp, deps, nd.n_dep == 0, &np_);
        if (!rc) {
          ++g->kinds[fp];
          rc = route_node(sc, i, specs[i], fam);
        }
        if (!rc) rc = add_kernel(specs[i], std::vector<cudaGraphNode_t>{np_}, false, &gn[i]);
      }
    } else {
      rc = route_node(nd, i, specs[i], fam);
      if (!rc) rc = add_kernel(specs[i], deps, nd.n_dep == 0, &gn[i]);
    }
    if (rc) {
      qtn_graph_destroy(g);
      return rc;
    }
    ++g->kinds[fam];
    g->node_kind.push_back(fam);
  }
  // optional result download after every kernel node
  if (io && io->d2h_bytes > 0) {
    cudaGraphNode_t d2h = nullptr;
    e = cudaGraphAddMemcpyNode1D(&d2h, g->graph, gn.data(), (size_t)n_nodes, io->d2h_dst, io->d2h_src,
                                 (size_t)io->d2h_bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      qtn_graph_destroy(g);
      return cuda_err(e, "cudaGraphAddMemcpyNode1D(d2h)");
    }
  }
  e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  if (e != cudaSuccess) {
    qtn_graph_destroy(g);
    return cuda_err(e, "cudaGraphInstantiate");
  }
  *out = g;
  return QTN_OK;
}

int qtn_graph_launch(qtn_graph_t* g, void* stream) {
  if (!g || !g->exec) return set_err(QTN_E_INVALID, "null graph");
  const cudaError_t e = cudaGraphLaunch(g->exec, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_err(e, "cudaGraphLaunch");
  return QTN_OK;
}

int qtn_graph_kinds(const qtn_graph_t* g, int32_t* counts) {
  if (!g || !counts) return set_err(QTN_E_INVALID, "null argument");
  for (int i = 0; i < 6; ++i) counts[i] = g->kinds[i];
  return QTN_OK;
}

int qtn_graph_node_kinds(const qtn_graph_t* g, int32_t* kinds, int32_t n) {
  if (!g || (n > 0 && !kinds)) return set_err(QTN_E_INVALID, "null argument");
  if (n != (int32_t)g->node_kind.size()) return set_err(QTN_E_INVALID, "graph has %d nodes, not %d",
                                                        (int)g->node_kind.size(), n);
  for (int i = 0; i < n; ++i) kinds[i] = g->node_kind[i];
  return QTN_OK;
}

int qtn_graph_destroy(qtn_graph_t* g) {
  if (!g) return QTN_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return QTN_OK;
}

int qtn_permute(int32_t src_dtype, const void* src, int64_t src_offset, int32_t dst_dtype, void* dst, int32_t rank,
                const int64_t* src_strides, void* stream) {
  if (!src || !dst) return set_err(QTN_E_INVALID, "null tensor");
  if (rank < 0 || rank > QTN_MAX_WIDTH) return set_err(QTN_E_UNSUPPORTED, "rank %d", rank);
  if (rank > 0 && !src_strides) return set_err(QTN_E_INVALID, "null strides");
  if ((src_dtype != QTN_C64 && src_dtype != QTN_C128) || (dst_dtype != QTN_C64 && dst_dtype != QTN_C128))
    return set_err(QTN_E_INVALID, "bad dtype");
  PermStrides st{};
  for (int j = 0; j < rank; ++j) st.s[j] = src_strides[j];
  const uint64_t n = 1ull << rank;
  const int threads = 256;
  const uint64_t blocks64 = (n + threads - 1) / threads;
  const int blocks = (int)(blocks64 > 148ull * 32 ? 148 * 32 : blocks64);
  cudaStream_t s = (cudaStream_t)stream;
  if (src_dtype == QTN_C128 && dst_dtype == QTN_C128)
    permute_kernel<double, double><<<blocks, threads, 0, s>>>((const double2*)src, src_offset, (double2*)dst, rank, st, n);
  else if (src_dtype == QTN_C128 && dst_dtype == QTN_C64)
    permute_kernel<double, float><<<blocks, threads, 0, s>>>((const double2*)src, src_offset, (float2*)dst, rank, st, n);
  else if (src_dtype == QTN_C64 && dst_dtype == QTN_C64)
    permute_kernel<float, float><<<blocks, threads, 0, s>>>((const float2*)src, src_offset, (float2*)dst, rank, st, n);
  else
    permute_kernel<float, double><<<blocks, threads, 0, s>>>((const float2*)src, src_offset, (double2*)dst, rank, st, n);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_err(e, "permute_kernel launch");
  return QTN_OK;
}

}  // extern "C"
