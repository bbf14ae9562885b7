// bucket_stream.cu — K5: the streaming-item kernel (one member carries every
// result bit).
//
// Same contraction as the reference's fast_kernel (src/tensor_core.py:148-164)
// for one program item, out[r] = sum_s prod_i m_i(r, s), for the items whose
// dominant member B carries ALL w result bits (SURVEY 8(d) class A, "reduce":
// B of rank w + k' is read once, the result is 2^k' times smaller).  Such an
// item is pure streaming: B once from HBM, the other members (a few MB at
// most) re-read from L1/L2, the result written once.  K1/K3/K4 stage the
// other members per tile through shared memory (a barrier and a bulk-copy
// round trip per tile); K5 reads every member directly:
//
//   tile   = 2^L consecutive results (L = 8 thread bits + VEC bit + the
//            per-thread step bits); the persistent grid walks the tiles
//   thread = results t*VEC + v + NT*VEC*u: lanes cover the fastest result
//            bits, so B (and any member carrying them) is read in contiguous
//            16-byte vectors, the output written in whole sectors
//   loads  = for UNR steps at once: every summed assignment s of every
//            loaded member (B with ld.global.cs — read once; the others with
//            __ldg — their elements are shared by the results they lack)
//   math   = acc = sum_s U[s] * prod_j x_j(s) in registers, s ascending; U[s]
//            = the product of the members that carry no result bit, once per
//            block
//
// Every index map is GF(2)-linear in the bits (member strides per bit), so
// offsets are sums of per-bit strides: thread part once, step part per step,
// tile part per tile.
#include "qtn_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>

int qtn_internal_set_error(int code, const char* msg);

#ifdef QTN_DEBUG
#define K5_CHECK(cond, ...)                                                        \
  do {                                                                             \
    if (!(cond)) {                                                                 \
      printf("K5_CHECK %s:%d (block %d thread %d): ", __FILE__, __LINE__,          \
             (int)blockIdx.x, (int)threadIdx.x);                                   \
      printf(__VA_ARGS__);                                                         \
      printf("\n");                                                               \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define K5_CHECK(cond, ...) \
  do {                      \
  } while (0)
#endif

namespace qtn_k5 {

constexpr int NT = 256;
constexpr int MAXM = QTN_MAX_MEMBERS;
constexpr int MAXV = 4;        // members loaded per result (B + up to 3)
constexpr int MAXKS = 3;       // summed bits
constexpr int MAXTB = 32;      // tile-selecting result bits
constexpr int MAXLB = 16;      // result bits inside a tile

struct Plan {
  void* out;
  const void* mptr[MAXM];      // loaded members first (B = 0), then uniform members
  int32_t nm, nv, k, w, L, b0, nsb;    // b0: first thread bit (1 = complex64 pairs); nsb: step bits (L = b0 + 8 + nsb)
  int32_t b_stream;            // B carries every result bit: read once, streaming loads (else re-read via L1/L2)
  int32_t pair[MAXV];          // c64: member j reads a (v = 0, 1) pair as one 16-byte vector
  int32_t bcast[MAXV];         // c64: member j does not carry result bit 0 (one value for the pair)
  int64_t n_tiles;
  int64_t span[MAXM];          // elements each member spans (QTN_DEBUG bounds checks)
  int64_t ts[MAXV + 1][MAXTB]; // stride of tile bit q (result bit L + q); index nv = output
  int32_t rs[MAXV][MAXLB];     // stride of tile-local result bit b
  int64_t ss[MAXM][MAXKS];     // stride of summed bit q
  unsigned long long* timing;
  int32_t item;
};

template <typename R> struct Cx;
template <> struct Cx<float> {
  using T = float2;
  using V = float4;
};
template <> struct Cx<double> {
  using T = double2;
  using V = double2;
};

template <typename T>
__device__ __forceinline__ T cmul(T a, T b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T>
__device__ __forceinline__ T cadd(T a, T b) {
  return {a.x + b.x, a.y + b.y};
}

__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ float2 ld_stream(const float2* p) { return __ldcs(p); }

// VEC = 2 (complex64 result pairs) or 1; NS = 2^k; NV = loaded members.
template <typename R, int VEC, int NS, int NV>
__device__ __forceinline__ void k5_body(const Plan& P) {
  using T = typename Cx<R>::T;
  using V = typename Cx<R>::V;
  constexpr int UNR = NS * NV * VEC <= 8 ? 2 : 1;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ T su[NS];
  __shared__ int64_t sof[NV][NS];   // member offsets of the summed assignments
  const int tid = threadIdx.x;
  // per-thread offsets of the thread bits (result bits b0 .. b0+7)
  int32_t th[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    int32_t o = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if ((tid >> b) & 1) o += P.rs[j][P.b0 + b];
    th[j] = o;
  }
  if (tid < NV * NS) {
    const int j = tid / NS, s = tid % NS;
    int64_t q = 0;
    for (int b = 0; b < P.k; ++b)
      if ((s >> b) & 1) q += P.ss[j][b];
    sof[j][s] = q;
  }
  int32_t tho = 0;   // output
#pragma unroll
  for (int b = 0; b < 8; ++b)
    if ((tid >> b) & 1) tho += 1 << (P.b0 + b);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  unsigned long long t_start = 0;
  if (P.timing && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  // U[s]: product of the members without result bits
  if (tid < NS) {
    T u = {R(1), R(0)};
    for (int j = NV; j < P.nm; ++j) {
      int64_t q = 0;
      for (int b = 0; b < P.k; ++b)
        if ((tid >> b) & 1) q += P.ss[j][b];
      K5_CHECK(q >= 0 && q < P.span[j], "uniform member %d element %lld", j, (long long)q);
      u = cmul(u, __ldg(reinterpret_cast<const T*>(P.mptr[j]) + q));
    }
    su[tid] = u;
  }
  __syncthreads();
  T U[NS];
  const bool has_u = P.nm > NV;
#pragma unroll
  for (int s = 0; s < NS; ++s) U[s] = su[s];
  const int nstep = 1 << P.nsb;
  const int sb0 = P.b0 + 8;   // first step bit
  for (int64_t h = blockIdx.x; h < P.n_tiles; h += gridDim.x) {
    int64_t tb[NV + 1];
#pragma unroll
    for (int j = 0; j <= NV; ++j) tb[j] = 0;
    for (int q = 0; q < P.w - P.L; ++q)
      if ((h >> q) & 1) {
#pragma unroll
        for (int j = 0; j < NV; ++j) tb[j] += P.ts[j][q];
        tb[NV] += P.ts[P.nv][q];
      }
    for (int u0 = 0; u0 < nstep; u0 += UNR) {
      // all loads of UNR steps first
      T x[UNR][NV][NS][VEC];
#pragma unroll
      for (int uu = 0; uu < UNR; ++uu) {
        const int u = u0 + uu < nstep ? u0 + uu : nstep - 1;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          int32_t uo = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b)
            if (b < P.nsb && ((u >> b) & 1)) uo += P.rs[j][sb0 + b];
          const T* base = reinterpret_cast<const T*>(P.mptr[j]) + tb[j] + th[j] + uo;
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const T* p = base + sof[j][s];
            K5_CHECK(p - reinterpret_cast<const T*>(P.mptr[j]) >= 0 &&
                         p - reinterpret_cast<const T*>(P.mptr[j]) + (VEC == 2 && !P.bcast[j] ? P.rs[j][0] : 0) <
                             P.span[j],
                     "member %d element %lld", j, (long long)(p - reinterpret_cast<const T*>(P.mptr[j])));
            if (VEC == 2) {
              if (P.pair[j]) {
                const V v = (j == 0 && P.b_stream) ? ld_stream(reinterpret_cast<const V*>(p)) : __ldg(reinterpret_cast<const V*>(p));
                const T* e = reinterpret_cast<const T*>(&v);
                x[uu][j][s][0] = e[0];
                x[uu][j][s][VEC - 1] = e[VEC - 1];
              } else if (P.bcast[j]) {
                x[uu][j][s][0] = __ldg(p);
                x[uu][j][s][VEC - 1] = x[uu][j][s][0];
              } else {
                x[uu][j][s][0] = __ldg(p);
                x[uu][j][s][VEC - 1] = __ldg(p + P.rs[j][0]);
              }
            } else {
              x[uu][j][s][0] = (j == 0 && P.b_stream) ? ld_stream(p) : __ldg(p);
            }
          }
        }
      }
#pragma unroll
      for (int uu = 0; uu < UNR; ++uu) {
        const int u = u0 + uu;
        if (u >= nstep) break;
        T acc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            T p = x[uu][0][s][v];
#pragma unroll
            for (int j = 1; j < NV; ++j) p = cmul(p, x[uu][j][s][v]);
            if (has_u) p = cmul(p, U[s]);
            acc[v] = s == 0 ? p : cadd(acc[v], p);
          }
        }
        const int64_t o = tb[NV] + tho + ((int64_t)u << sb0);
        K5_CHECK(o >= 0 && o + VEC <= ((int64_t)1 << P.w), "result %lld", (long long)o);
        T* op = reinterpret_cast<T*>(P.out) + o;
        if (VEC == 2) {
          V w;
          T* we = reinterpret_cast<T*>(&w);
          we[0] = acc[0];
          we[VEC - 1] = acc[VEC - 1];
          *reinterpret_cast<V*>(op) = w;
        } else {
          *op = acc[0];
        }
      }
    }
  }
  if (P.timing && tid == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    atomicMin(&P.timing[2 * P.item], t_start);
    atomicMax(&P.timing[2 * P.item + 1], t_end);
  }
}

template <int NS, int NV>
__global__ void __launch_bounds__(NT, 2) k5_kernel_c64(const __grid_constant__ Plan P) {
  k5_body<float, 2, NS, NV>(P);
}
template <int NS, int NV>
__global__ void __launch_bounds__(NT, 2) k5_kernel_c128(const __grid_constant__ Plan P) {
  k5_body<double, 1, NS, NV>(P);
}

template <int NS>
const void* fn_nv(bool c64, int nv) {
  switch (nv) {
    case 1: return c64 ? (const void*)k5_kernel_c64<NS, 1> : (const void*)k5_kernel_c128<NS, 1>;
    case 2: return c64 ? (const void*)k5_kernel_c64<NS, 2> : (const void*)k5_kernel_c128<NS, 2>;
    case 3: return c64 ? (const void*)k5_kernel_c64<NS, 3> : (const void*)k5_kernel_c128<NS, 3>;
    default: return c64 ? (const void*)k5_kernel_c64<NS, 4> : (const void*)k5_kernel_c128<NS, 4>;
  }
}

const void* fn_of(bool c64, int k, int nv) {
  if (k == 1) return fn_nv<2>(c64, nv);
  if (k == 2) return fn_nv<4>(c64, nv);
  return fn_nv<8>(c64, nv);
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

// Plan K5 for `d`: QTN_E_UNSUPPORTED unless one member carries every result
// bit (or, max_e > 0, all but at most max_e of them: the dominant member is
// then re-read through L1/L2 once per missing-bit assignment) and at most
// MAXV members carry result bits.
int make_plan(const qtn_bucket_desc_t* d, int max_e, Plan* P) {
  memset(P, 0, sizeof(*P));
  const int w = d->w, k = d->k, nm = d->n_mem;
  if (d->dtype != QTN_C64 && d->dtype != QTN_C128) return fail(QTN_E_INVALID, "K5: bad dtype");
  const bool c64 = d->dtype == QTN_C64;
  const int vec = c64 ? 2 : 1;
  const int vb = c64 ? 1 : 0;
  if (k < 1 || k > MAXKS || nm < 1 || nm > MAXM || w < vb + 8 || w > 40)
    return fail(QTN_E_UNSUPPORTED, "K5: w=%d k=%d n_mem=%d", w, k, nm);
  // dominant member: the most result bits (the first such member)
  int iB = -1, best = -1;
  for (int i = 0; i < nm; ++i) {
    int c = 0;
    for (int b = 0; b < w; ++b) c += d->mem[i].strides[b] != 0;
    if (c > best) best = c, iB = i;
  }
  if (best < w - max_e) return fail(QTN_E_UNSUPPORTED, "K5: no member carries every result bit");
  P->b_stream = best == w ? 1 : 0;
  // loaded members: B first, then the others with result bits (member order)
  int ord[MAXM], nv = 0, nmo = 0;
  ord[nv++] = iB;
  for (int i = 0; i < nm; ++i) {
    if (i == iB) continue;
    bool any = false;
    for (int b = 0; b < w; ++b) any |= d->mem[i].strides[b] != 0;
    if (any) ord[nv++] = i;
  }
  if (nv > MAXV) return fail(QTN_E_UNSUPPORTED, "K5: %d members carry result bits", nv);
  nmo = nv;
  for (int i = 0; i < nm; ++i) {
    bool any = false;
    for (int b = 0; b < w; ++b) any |= d->mem[i].strides[b] != 0;
    if (!any) ord[nmo++] = i;
  }
  const size_t esz = c64 ? 8 : 16;
  for (int j = 0; j < nm; ++j) {
    const qtn_bmember_t& m = d->mem[ord[j]];
    if (!m.data) return fail(QTN_E_INVALID, "K5: null member %d", ord[j]);
    int64_t span = 1;
    for (int b = 0; b < w + k; ++b) {
      if (m.strides[b] < 0) return fail(QTN_E_UNSUPPORTED, "K5: negative stride");
      span += m.strides[b];
    }
    P->mptr[j] = m.data;
    P->span[j] = span;
    for (int q = 0; q < k; ++q) P->ss[j][q] = m.strides[w + q];
  }
  if (!d->out) return fail(QTN_E_INVALID, "K5: null output");
  // tile: vec bit + 8 thread bits + up to 2 step bits (1024 complex128 / 2048 complex64 results)
  const int nsb = std::min(2, w - vb - 8);
  const int L = vb + 8 + nsb;
  if (w - L > MAXTB || L > MAXLB) return fail(QTN_E_UNSUPPORTED, "K5: w=%d", w);
  for (int j = 0; j < nv; ++j) {
    const qtn_bmember_t& m = d->mem[ord[j]];
    for (int b = 0; b < L; ++b) {
      if (m.strides[b] >= ((int64_t)1 << 31)) return fail(QTN_E_UNSUPPORTED, "K5: tile stride");
      P->rs[j][b] = (int32_t)m.strides[b];
    }
    for (int q = 0; q < w - L; ++q) P->ts[j][q] = m.strides[L + q];
    if (c64) {
      // pair loads need the v pair adjacent and 16-byte aligned
      bool ok = m.strides[0] == 1 && ((uintptr_t)m.data % 16) == 0;
      for (int b = 1; b < w + k && ok; ++b) ok = m.strides[b] % 2 == 0;
      P->pair[j] = ok ? 1 : 0;
      P->bcast[j] = m.strides[0] == 0 ? 1 : 0;
    }
  }
  if (((uintptr_t)d->out % 16) != 0) return fail(QTN_E_UNSUPPORTED, "K5: output not 16-byte aligned");
  for (int q = 0; q < w - L; ++q) P->ts[nv][q] = (int64_t)1 << (L + q);
  P->out = d->out;
  P->nm = nm;
  P->nv = nv;
  P->k = k;
  P->w = w;
  P->L = L;
  P->b0 = vb;
  P->nsb = nsb;
  P->n_tiles = (int64_t)1 << (w - L);
  (void)vec;
  (void)esz;
  return QTN_OK;
}

}  // namespace qtn_k5

size_t qtn_k5_plan_bytes() { return sizeof(qtn_k5::Plan); }

// Program-graph node for one item (qtn_graph_create_host): QTN_E_UNSUPPORTED
// when no member carries every result bit.
int qtn_k5_node(const qtn_bucket_desc_t* d, int max_e, unsigned long long* timing, int32_t item, void* plan,
                const void** fn, int* grid, int* smem) {
  using namespace qtn_k5;
  Plan* P = reinterpret_cast<Plan*>(plan);
  int rc = make_plan(d, max_e, P);
  if (rc) return rc;
  P->timing = timing;
  P->item = item;
  *fn = fn_of(d->dtype == QTN_C64, P->k, P->nv);
  *smem = 0;
  int per_sm = 0;
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, *fn, NT, 0);
  if (e != cudaSuccess) return fail(QTN_E_CUDA, "occupancy: %s", cudaGetErrorString(e));
  if (per_sm < 1) return fail(QTN_E_UNSUPPORTED, "K5 cannot be resident");
  *grid = (int)std::min<int64_t>(P->n_tiles, (int64_t)per_sm * sm_count());
  return QTN_OK;
}

extern "C" int qtn_bucket_stream(const qtn_bucket_desc_t* d, void* stream) {
  using namespace qtn_k5;
  if (!d) return fail(QTN_E_INVALID, "null descriptor");
  static thread_local Plan P;
  const void* fn = nullptr;
  int grid = 0, smem = 0;
  int rc = qtn_k5_node(d, 0, nullptr, 0, &P, &fn, &grid, &smem);
  if (rc) return rc;
  void* args[] = {&P};
  const cudaError_t e = cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(NT), args, 0, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(QTN_E_CUDA, "K5 launch: %s", cudaGetErrorString(e));
  return QTN_OK;
}
