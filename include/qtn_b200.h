/*
 * qtn_b200.h — C ABI of the B200 bucket-elimination engine (libqtn_b200.so).
 *
 * The reference (qtnsim, pure Python/NumPy) has no native boundary; its
 * process-bucket / get-result seam is the Python call
 *     contract_bucket(Bucket, Backend)        src/tensor_core.py:167-188
 * invoked from the elimination loop of
 *     contract_network(tn, order, backend)    src/ordering.py:148-189
 * (paths relative to /root/reference/pkg/).  This ABI is what a binding for
 * that seam calls (see INTEGRATION.md for the ctypes stub): the host plans a
 * "program" (buckets, members, dependencies, arena offsets) from the
 * symbolic dry run (src/ordering.py:97-145) and launches it here; every
 * buffer is owned by the caller (PyTorch), passed as a plain device pointer.
 *
 * Conventions
 *  - Status: int, 0 = QTN_OK, negative = QTN_E_*; details in qtn_last_error()
 *    (thread-local).  No exceptions cross the ABI.
 *  - Element types: complex64 (float2) or complex128 (double2), QTN_C64/QTN_C128.
 *  - Canonical layout: every tensor in a program is stored with its axes
 *    sorted by elimination position, earliest-eliminated axis SLOWEST.  A
 *    member of bucket b therefore has b as its slowest axis and its other
 *    axes in the same relative order as the bucket's result axes, so its
 *    element offset is   b * 2^popc(mask) + pext(r, mask)   for result
 *    element r, where bit j of `mask` says the member carries result axis j
 *    (j = 0 is the fastest result axis).
 *  - Thread safety: launches on distinct streams are independent; a program's
 *    control block must not be shared by concurrent launches.
 */
#ifndef QTN_B200_H
#define QTN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QTN_ABI_VERSION 1

enum {
  QTN_OK = 0,
  QTN_E_INVALID = -1,     /* bad descriptor / argument   (reference: ValueError) */
  QTN_E_CUDA = -2,        /* CUDA runtime error (message in qtn_last_error)    */
  QTN_E_UNSUPPORTED = -3, /* shape or dtype outside what the kernels support   */
  QTN_E_NODEVICE = -4     /* no CUDA device visible                            */
};

enum { QTN_C64 = 0, QTN_C128 = 1 };

/* Largest number of members a bucket may have (reference buckets at the
 * BASELINE configs have 1-6; larger buckets are split by the planner). */
#define QTN_MAX_MEMBERS 8
/* Largest result width a bucket may have (2^40 elements). */
#define QTN_MAX_WIDTH 40

/* One member tensor of one bucket (16 bytes). */
typedef struct {
  uint64_t off;  /* element offset of the member in the arena            */
  uint64_t mask; /* result-axis coverage, bit j = result axis j (j=0 fastest) */
} qtn_member_t;

/* One work item: a bucket contraction (w >= 0) or an instance finaliser
 * (w == QTN_FINALIZE) that multiplies rank-0 values into a result slot —
 * the get-result step (src/ordering.py:167-170,183-184).  48 bytes. */
#define QTN_FINALIZE (-1)
typedef struct {
  uint64_t out_off;   /* element offset of the result in the arena          */
  int32_t w;          /* result rank, or QTN_FINALIZE                       */
  int32_t tile_bits;  /* L: each tile computes 2^L consecutive results      */
  int32_t mem_begin;  /* first member in the member table                   */
  int32_t n_mem;      /* 1..QTN_MAX_MEMBERS (finaliser: any count >= 0)     */
  int32_t dep_begin;  /* first dependency in the dependency table           */
  int32_t n_dep;
  int32_t tick_begin; /* first ticket; tickets of a program are dense       */
  int32_t n_tiles;    /* 2^(w - L); 1 for a finaliser                       */
  int32_t slot;       /* finaliser: result slot (double2); else -1          */
  int32_t smem_elems; /* staged elements per tile (<= program smem budget)  */
} qtn_bucket_t;

/* Dependency: wait until bucket `bucket` has completed `need` tiles. */
typedef struct {
  int32_t bucket;
  int32_t need;
} qtn_dep_t;

/* A planned program (one or many lightcones / slices).  All pointers are
 * DEVICE pointers owned by the caller.  `tick_begin` must be a dense int32
 * copy of buckets[i].tick_begin (used for ticket -> bucket search). */
typedef struct {
  int32_t dtype;                /* QTN_C64 / QTN_C128                         */
  int32_t n_buckets;
  int32_t n_tickets;
  int32_t smem_bytes;           /* dynamic shared memory per block (staging)  */
  int32_t grid;                 /* 0 = all resident blocks (occupancy)        */
  int32_t flags;                /* reserved, 0                                */
  const qtn_bucket_t* buckets;
  const qtn_member_t* members;
  const qtn_dep_t* deps;
  const int32_t* tick_begin;
  uint32_t* ctrl;               /* 2 + n_buckets words, zero before 1st launch */
  void* arena;                  /* element storage (16-byte aligned); NULL =
                                   offsets are absolute addresses / elem size  */
  double* results;              /* 2 doubles per finaliser slot               */
  unsigned long long* timing;   /* optional: 2 per bucket (first start, last end, ns) */
} qtn_program_t;

/* ABI version (QTN_ABI_VERSION). */
int qtn_abi_version(void);
/* Last error message of the calling thread ("" if none). */
const char* qtn_last_error(void);
/* Number of visible CUDA devices (0 on a CPU-only host; never fails). */
int qtn_device_count(int* count);
/* Resident blocks of the program kernel for dtype/smem on the current device. */
int qtn_program_grid(int32_t dtype, int32_t smem_bytes, int32_t* grid_out);
/* Zero the control block (tickets, exit count, per-bucket completion). */
int qtn_program_reset(const qtn_program_t* prog, void* stream);
/* Launch the persistent program kernel on `stream` (cudaStream_t, may be 0).
 * The kernel leaves the control block zeroed on exit, so launches of the
 * same program can be issued back to back (or captured in a CUDA graph). */
int qtn_program_launch(const qtn_program_t* prog, void* stream);
/* dst[e] = convert(src[sum_j bit_j(e) * src_strides[j]]) for e < 2^rank,
 * j = 0 the fastest dst axis; src/dst element types given separately
 * (complex128 -> complex64 narrowing allowed).  General axis permutation +
 * slice offset for tensors entering a program in a non-canonical layout
 * (src/tensor_core.py:107-114, src/ordering.py:233-248). */
int qtn_permute(int32_t src_dtype, const void* src, int64_t src_offset,
                int32_t dst_dtype, void* dst, int32_t rank,
                const int64_t* src_strides, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* QTN_B200_H */
