// k4_plan.h — the K4 tile plan (csrc/bucket_expand.cu), shared with K6
// (csrc/bucket_fused.cu): constants, the Plan record passed to the kernels as
// a __grid_constant__ parameter, complex helpers and the planner entry.
#ifndef QTN_K4_PLAN_H
#define QTN_K4_PLAN_H

#include "qtn_b200.h"

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

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

// planner (host): K4 tile plan of descriptor d; nq > 0 sets the top nq result
// fail(): set the thread's error message, return code.
// bits aside (K6); at most ne_max B-lacking bits become expansion bits (the
// others tile bits: smaller tiles, B read once per tile); ntb thread bits
// (K6 lane-split plans use 7: the 8th thread bit splits the q runs).
int make_plan(const qtn_bucket_desc_t* d, int min_e, Plan* P, int* smem, int nq = 0, int ne_max = MAXE,
              int ntb = TBB);
int fail(int code, const char* fmt, ...);
int sm_count();

}  // namespace qtn_k4

#endif  // QTN_K4_PLAN_H
