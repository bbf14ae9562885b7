// qtn_b200.cu — sm_100a kernels + C ABI of the bucket-elimination engine.
//
// One persistent "program" kernel executes a whole planned elimination
// (one lightcone, one slice, or a batch of them) in a single launch:
//
//  * Work is a dense ticket space: bucket i owns tickets
//    [tick_begin_i, tick_begin_i + n_tiles_i); buckets appear in a
//    topological order of the bucket in-tree (src/ordering.py:175-187), so a
//    block that takes a ticket only ever waits on LOWER tickets.  Tickets are
//    taken by running blocks (atomicAdd), which makes the schedule
//    deadlock-free whatever the residency.
//  * A tile is 2^L consecutive result elements of one bucket.  Its members
//    are either STREAMED (the member carries all L tile axes: two contiguous
//    2^L runs, b = 0 and b = 1, read with 16-byte vector loads straight from
//    HBM/L2) or STAGED (the member carries a subset of the tile axes: its two
//    contiguous 2^popc runs are copied to shared memory once per tile and
//    gathered with a precomputed pext table).
//  * out[r] = prod_i T_i[b=0] + prod_i T_i[b=1] — the reference's
//    fast_kernel product order (src/tensor_core.py:148-164): members in
//    bucket order, then b = 0 + b = 1.
//  * Completion is a per-bucket tile counter (release: __syncthreads +
//    __threadfence + atomicAdd; acquire: ld.acquire.gpu spin).  Data produced
//    inside the launch is read with ld.global.cg (L2, never a stale L1 line).
//  * Finaliser items multiply an instance's rank-0 values in double precision
//    into a result slot: the get-result scalar (src/ordering.py:167-170,183-184).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo ...
#include "qtn_b200.h"

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>

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

constexpr int NT = 256;                 // threads per block
constexpr int MAXM = QTN_MAX_MEMBERS;   // members per bucket
constexpr int MAXS = 16;                // vector steps per tile: 2^L / (VEC * NT)

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

// vector <-> element views
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
__device__ __forceinline__ uint64_t pext64(uint64_t x, uint64_t m) {
  uint64_t r = 0;
  for (int k = 0; m; ++k) {
    const uint64_t low = m & (0ull - m);
    if (x & low) r |= 1ull << k;
    m ^= low;
  }
  return r;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Per-block view of the bucket being processed (shared memory).
struct BlockCtx {
  qtn_bucket_t b;
  uint64_t off[MAXM];    // member element offset in arena
  uint64_t mhi[MAXM];    // member mask >> L
  uint64_t bstr[MAXM];   // b stride = 2^popc(mask)
  uint64_t base[MAXM];   // b = 0 offset of the member's run for this tile
  uint32_t mlo[MAXM];    // member mask & (2^L - 1)
  int32_t pclo[MAXM];    // popc(mlo)
  int32_t seg[MAXM];     // staged: smem element offset of the run pair; streamed: -1
  int32_t seglen[MAXM];  // staged: 2^pclo
  int32_t gs[MAXM][MAXS];  // pext(VEC*NT*s, mlo)
  int32_t bucket;
  int32_t tick;
  int32_t next;
  int32_t last;
};

template <typename R>
__global__ void __launch_bounds__(NT) program_kernel(const qtn_program_t P) {
  using T = typename Cx<R>::T;
  using V = typename Cx<R>::V;
  constexpr int VEC = Cx<R>::VEC;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sseg = reinterpret_cast<T*>(smem_raw);
  __shared__ BlockCtx S;

  T* A = reinterpret_cast<T*>(P.arena);
  uint32_t* done = P.ctrl + 2;
  const int tid = threadIdx.x;

  int cur = 0;         // bucket of the current ticket (block-uniform, monotone)
  int prepared = -1;   // bucket whose per-bucket tables are loaded in S
  int gt[MAXM];        // per-thread pext(VEC*tid, mlo_i)

  if (tid == 0) S.next = (int)atomicAdd(&P.ctrl[0], 1u);
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      S.tick = S.next;
      // prefetch the following ticket; its latency overlaps this tile
      if (S.tick < P.n_tickets) S.next = (int)atomicAdd(&P.ctrl[0], 1u);
    }
    __syncthreads();
    const int tk = S.tick;
    if (tk >= P.n_tickets) break;

    // ---- ticket -> bucket: 32-ary search over tick_begin[cur..] (warp 0) ----
    if (tid < 32) {
      int lo = cur, hi = P.n_buckets - 1;
      if (lo < hi && __ldg(&P.tick_begin[lo + 1]) > tk) hi = lo;  // same bucket
      while (hi > lo) {
        const int span = hi - lo;
        const int step = (span + 31) / 32;
        int p = lo + (tid + 1) * step;
        if (p > hi) p = hi;
        const bool ok = __ldg(&P.tick_begin[p]) <= tk;
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        const int c = __popc(bal);   // predicate is monotone: a prefix of lanes
        if (c == 0) {
          hi = lo + step - 1;
        } else {
          const int plast = min(lo + c * step, hi);
          const int pnext = lo + (c + 1) * step;
          lo = plast;
          if (c < 32 && pnext - 1 < hi) hi = pnext - 1;
        }
      }
      if (tid == 0) S.bucket = lo;
    }
    __syncthreads();
    cur = S.bucket;

    // ---- per-bucket preparation (once per bucket per block) ----
    if (cur != prepared) {
      if (tid == 0) S.b = P.buckets[cur];
      __syncthreads();
      const int nm = S.b.w >= 0 ? S.b.n_mem : 0;
      const int L = S.b.tile_bits;
      // wait for producers (and WAR predecessors)
      for (int k = tid; k < S.b.n_dep; k += NT) {
        const qtn_dep_t d = P.deps[S.b.dep_begin + k];
        const uint32_t* c = done + d.bucket;
        while (ld_acquire(c) < (uint32_t)d.need) __nanosleep(64);
      }
      if (tid < nm) {
        const qtn_member_t m = P.members[S.b.mem_begin + tid];
        const uint32_t lowmask = (L >= 32) ? 0xffffffffu : ((1u << L) - 1u);
        S.off[tid] = m.off;
        S.mlo[tid] = (uint32_t)(m.mask & lowmask);
        S.mhi[tid] = m.mask >> L;
        S.pclo[tid] = __popc((uint32_t)(m.mask & lowmask));
        S.bstr[tid] = 1ull << __popcll(m.mask);
        S.seglen[tid] = 1 << S.pclo[tid];
      }
      __syncthreads();
      if (tid == 0) {
        int acc = 0;
        for (int i = 0; i < nm; ++i) {
          if (S.pclo[i] == L) {
            S.seg[i] = -1;
          } else {
            S.seg[i] = acc;
            acc += 2 * S.seglen[i];
          }
        }
      }
      if (tid < nm * MAXS) {
        const int i = tid / MAXS, s = tid % MAXS;
        S.gs[i][s] = (int)pext32((uint32_t)(VEC * NT * s), S.mlo[i]);
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < MAXM; ++i) gt[i] = (i < nm) ? (int)pext32((uint32_t)(VEC * tid), S.mlo[i]) : 0;
      prepared = cur;
    }

    const int h = tk - S.b.tick_begin;
    unsigned long long t_start = 0;
    if (P.timing && tid == 0) t_start = globaltimer();

    if (S.b.w < 0) {
      // ---- finaliser: product of rank-0 values, in double, member order ----
      if (tid == 0) {
        double re = 1.0, im = 0.0;
        for (int i = 0; i < S.b.n_mem; ++i) {
          const qtn_member_t m = P.members[S.b.mem_begin + i];
          const T v = __ldcg(A + m.off);
          const double vr = (double)v.x, vi = (double)v.y;
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
      const int nelem = 1 << L;
      if (tid < nm) S.base[tid] = S.off[tid] + (pext64((uint64_t)h, S.mhi[tid]) << S.pclo[tid]);
      __syncthreads();
      // stage partial-coverage members (two contiguous runs each) into smem
      for (int i = 0; i < nm; ++i) {
        const int sg = S.seg[i];
        if (sg < 0) continue;
        const int len = S.seglen[i];
        const T* src0 = A + S.base[i];
        const T* src1 = src0 + S.bstr[i];
        for (int q = tid; q < 2 * len; q += NT)
          sseg[sg + q] = __ldcg(q < len ? src0 + q : src1 + (q - len));
      }
      __syncthreads();
      T* out = A + S.b.out_off + (uint64_t)h * (uint64_t)nelem;
      if (nelem >= VEC * NT) {
        const int ns = nelem / (VEC * NT);
        for (int s = 0; s < ns; ++s) {
          const int e0 = VEC * (tid + NT * s);
          T p0[VEC], p1[VEC];
#pragma unroll
          for (int i = 0; i < MAXM; ++i) {
            if (i >= nm) break;
            T x0[VEC], x1[VEC];
            if (S.seg[i] < 0) {
              const V* v0 = reinterpret_cast<const V*>(A + S.base[i] + e0);
              const V* v1 = reinterpret_cast<const V*>(A + S.base[i] + S.bstr[i] + e0);
              split(__ldcg(v0), x0);
              split(__ldcg(v1), x1);
            } else {
              const int idx = gt[i] + S.gs[i][s];
              const T* s0 = sseg + S.seg[i];
              const T* s1 = s0 + S.seglen[i];
              const int bit0 = (int)(S.mlo[i] & 1u);
#pragma unroll
              for (int v = 0; v < VEC; ++v) {
                x0[v] = s0[idx + (v & bit0)];
                x1[v] = s1[idx + (v & bit0)];
              }
            }
            if (i == 0) {
#pragma unroll
              for (int v = 0; v < VEC; ++v) { p0[v] = x0[v]; p1[v] = x1[v]; }
            } else {
#pragma unroll
              for (int v = 0; v < VEC; ++v) { p0[v] = cmul(p0[v], x0[v]); p1[v] = cmul(p1[v], x1[v]); }
            }
          }
          T r[VEC];
#pragma unroll
          for (int v = 0; v < VEC; ++v) r[v] = cadd(p0[v], p1[v]);
          *reinterpret_cast<V*>(out + e0) = join(r);
        }
      } else {
        for (int e = tid; e < nelem; e += NT) {
          T p0, p1;
          for (int i = 0; i < nm; ++i) {
            T x0, x1;
            if (S.seg[i] < 0) {
              x0 = __ldcg(A + S.base[i] + e);
              x1 = __ldcg(A + S.base[i] + S.bstr[i] + e);
            } else {
              const int idx = (int)pext32((uint32_t)e, S.mlo[i]);
              x0 = sseg[S.seg[i] + idx];
              x1 = sseg[S.seg[i] + S.seglen[i] + idx];
            }
            if (i == 0) {
              p0 = x0;
              p1 = x1;
            } else {
              p0 = cmul(p0, x0);
              p1 = cmul(p1, x1);
            }
          }
          out[e] = cadd(p0, p1);
        }
      }
    }

    // ---- publish completion of this tile ----
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(&done[cur], 1u);
      if (P.timing) {
        atomicMin(&P.timing[2 * cur], t_start);
        atomicMax(&P.timing[2 * cur + 1], globaltimer());
      }
    }
  }

  // ---- exit: the last block out leaves the control block zeroed ----
  if (tid == 0) {
    const unsigned v = atomicAdd(&P.ctrl[1], 1u);
    S.last = (v == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (S.last) {
    __threadfence();
    for (int i = tid; i < P.n_buckets; i += NT) done[i] = 0u;
    if (tid == 0) {
      P.ctrl[0] = 0u;
      P.ctrl[1] = 0u;
    }
  }
}

struct PermStrides {
  int64_t s[QTN_MAX_WIDTH + 4];
};

template <typename RS, typename RD>
__global__ void permute_kernel(const typename Cx<RS>::T* __restrict__ src, int64_t src_off,
                               typename Cx<RD>::T* __restrict__ dst, int rank, PermStrides st,
                               uint64_t n) {
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

template <typename R>
int configure_program(int smem) {
  const cudaError_t e = cudaFuncSetAttribute(program_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_err(e, "cudaFuncSetAttribute(program_kernel)");
  return QTN_OK;
}

template <typename R>
int grid_for(int smem, int* grid) {
  int dev = 0, nsm = 0, nb = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_err(e, "cudaGetDevice");
  e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_err(e, "cudaDeviceGetAttribute");
  int rc = configure_program<R>(smem);
  if (rc) return rc;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, program_kernel<R>, NT, smem);
  if (e != cudaSuccess) return cuda_err(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  if (nb < 1) return set_err(QTN_E_UNSUPPORTED, "program kernel cannot be resident with %d B smem", smem);
  *grid = nb * nsm;
  return QTN_OK;
}

int check_program(const qtn_program_t* p) {
  if (!p) return set_err(QTN_E_INVALID, "null program");
  if (p->dtype != QTN_C64 && p->dtype != QTN_C128) return set_err(QTN_E_INVALID, "bad dtype %d", p->dtype);
  if (p->n_buckets < 0 || p->n_tickets < 0) return set_err(QTN_E_INVALID, "negative sizes");
  // arena may be NULL: member/result offsets are then absolute addresses / element size
  if (p->n_buckets > 0 && (!p->buckets || !p->tick_begin || !p->ctrl))
    return set_err(QTN_E_INVALID, "null device table");
  if (p->smem_bytes < 0 || p->smem_bytes > 227 * 1024) return set_err(QTN_E_INVALID, "smem_bytes %d", p->smem_bytes);
  return QTN_OK;
}

}  // namespace

extern "C" {

int qtn_abi_version(void) { return QTN_ABI_VERSION; }

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

int qtn_program_grid(int32_t dtype, int32_t smem_bytes, int32_t* grid_out) {
  if (!grid_out) return set_err(QTN_E_INVALID, "null grid_out");
  int g = 0;
  const int rc = dtype == QTN_C64 ? grid_for<float>(smem_bytes, &g) : grid_for<double>(smem_bytes, &g);
  if (rc) return rc;
  *grid_out = g;
  return QTN_OK;
}

int qtn_program_reset(const qtn_program_t* p, void* stream) {
  int rc = check_program(p);
  if (rc) return rc;
  const cudaError_t e = cudaMemsetAsync(p->ctrl, 0, sizeof(uint32_t) * (2 + (size_t)p->n_buckets),
                                        (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_err(e, "cudaMemsetAsync(ctrl)");
  return QTN_OK;
}

int qtn_program_launch(const qtn_program_t* p, void* stream) {
  int rc = check_program(p);
  if (rc) return rc;
  if (p->n_tickets == 0) return QTN_OK;
  int grid = p->grid;
  if (grid <= 0) {
    rc = qtn_program_grid(p->dtype, p->smem_bytes, &grid);
    if (rc) return rc;
  } else {
    rc = p->dtype == QTN_C64 ? configure_program<float>(p->smem_bytes) : configure_program<double>(p->smem_bytes);
    if (rc) return rc;
  }
  if (p->dtype == QTN_C64)
    program_kernel<float><<<grid, NT, p->smem_bytes, (cudaStream_t)stream>>>(*p);
  else
    program_kernel<double><<<grid, NT, p->smem_bytes, (cudaStream_t)stream>>>(*p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_err(e, "program_kernel launch");
  return QTN_OK;
}

int qtn_permute(int32_t src_dtype, const void* src, int64_t src_offset, int32_t dst_dtype, void* dst,
                int32_t rank, const int64_t* src_strides, void* stream) {
  if (!src || !dst) return set_err(QTN_E_INVALID, "null tensor");
  if (rank < 0 || rank > QTN_MAX_WIDTH) return set_err(QTN_E_UNSUPPORTED, "rank %d", rank);
  if (rank > 0 && !src_strides) return set_err(QTN_E_INVALID, "null strides");
  if ((src_dtype != QTN_C64 && src_dtype != QTN_C128) || (dst_dtype != QTN_C64 && dst_dtype != QTN_C128))
    return set_err(QTN_E_INVALID, "bad dtype");
  PermStrides st{};
  for (int j = 0; j < rank; ++j) st.s[j] = src_strides[j];
  const uint64_t n = 1ull << rank;
  const int threads = 256;
  uint64_t blocks64 = (n + threads - 1) / threads;
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
