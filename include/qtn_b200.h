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
 *    sorted by elimination position, earliest-eliminated axis SLOWEST.
 *  - A work item sums k >= 1 indices at once (k = 1 is one reference bucket;
 *    k > 1 is a chain of reference buckets merged by the planner — the
 *    intermediate results never touch HBM).  The summed indices are all
 *    eliminated before any result index, so a member's summed axes are its
 *    slowest axes and its element offset is
 *        (pext(s, smask) << popc(mask)) + pext(r, mask)
 *    for summed assignment s (k bits) and result element r (w bits); bit j
 *    of `mask` / `smask` says the member carries result / summed axis j
 *    (j = 0 is the fastest, i.e. latest-eliminated, axis).
 *    out[r] = sum_{s = 0 .. 2^k - 1} prod_i member_i(s, r), s ascending.
 *  - Thread safety: launches on distinct streams are independent; a program's
 *    control block must not be shared by concurrent launches.
 */
#ifndef QTN_B200_H
#define QTN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QTN_ABI_VERSION 10

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
/* Largest number of indices one work item sums (merged bucket chain). */
#define QTN_MAX_SUMMED 6

/* Member classes for the large-item kernels (chosen by the planner from the
 * item's tile bits L and step mask): */
enum {
  QTN_CLS_STREAMED = 0,  /* carries every tile bit: 16-byte loads from HBM/L2   */
  QTN_CLS_UNIFORM = 1,   /* carries no tile bit: folded into U[s] once per tile */
  QTN_CLS_INVARIANT = 2, /* none of the step bits: folded into P[s] (k == 1)    */
  QTN_CLS_VARYING = 3    /* staged run in smem, gathered per step              */
};

/* One member tensor of one work item (24 bytes). */
typedef struct {
  uint64_t off;   /* element offset of the member in the arena             */
  uint64_t mask;  /* result-axis coverage, bit j = result axis j (j=0 fastest) */
  uint32_t smask; /* summed-axis coverage (k bits)                         */
  uint32_t cls;   /* QTN_CLS_* (large items)                               */
} qtn_member_t;

/* One work item: a (merged) bucket contraction (w >= 0) or an instance
 * finaliser (w == QTN_FINALIZE) that multiplies rank-0 values into a result
 * slot — the get-result step (src/ordering.py:167-170,183-184).  64 bytes. */
#define QTN_FINALIZE (-1)
typedef struct {
  uint64_t out_off;   /* element offset of the result in the arena          */
  int32_t w;          /* result rank, or QTN_FINALIZE                       */
  int32_t tile_bits;  /* L: each tile computes 2^L consecutive results      */
  int32_t k;          /* summed indices, 1..QTN_MAX_SUMMED                  */
  int32_t mem_begin;  /* first member in the member table                   */
  int32_t n_mem;      /* 1..QTN_MAX_MEMBERS (finaliser: any count >= 0)     */
  int32_t dep_begin;  /* first dependency in the dependency table           */
  int32_t n_dep;
  int32_t tick_begin; /* first ticket; tickets of a program are dense       */
  int32_t n_tiles;    /* 2^(w - L); 1 for a finaliser                       */
  int32_t slot;       /* finaliser: result slot (double2); else -1          */
  int32_t smem_elems; /* staged elements per tile (<= program smem budget)  */
  uint32_t stmask;    /* tile bits each thread walks sequentially (vector
                         path; 0 = default).  Members not carrying any of
                         them are multiplied once per tile and reused.       */
  int32_t reserved[2];
} qtn_bucket_t;

/* Dependency: wait until bucket `bucket` has completed `need` tiles. */
typedef struct {
  int32_t bucket;
  int32_t need;
} qtn_dep_t;

/* A planned program (one or many lightcones / slices).  All pointers are
 * DEVICE pointers owned by the caller.  `tick_begin` must be a dense int32
 * copy of buckets[i].tick_begin (stage-relative tickets of small items, used
 * for ticket -> item search).  ctrl = 2 words per graph node (small-stage
 * ticket and exit counters) followed by one completion counter per item. */
typedef struct {
  int32_t dtype;                /* QTN_C64 / QTN_C128                         */
  int32_t n_buckets;
  int32_t n_tickets;
  int32_t smem_bytes;           /* dynamic shared memory per block (staging)  */
  int32_t grid;                 /* K2 stages: 0 = all resident blocks; > 0 caps
                                   the persistent grid (schedule tests)        */
  int32_t n_nodes;              /* graph nodes (ctrl layout, see above)       */
  const qtn_bucket_t* buckets;
  const qtn_member_t* members;
  const qtn_dep_t* deps;
  const int32_t* tick_begin;
  uint32_t* ctrl;               /* 2 + n_buckets words, zero before 1st launch */
  void* arena;                  /* element storage (16-byte aligned); NULL =
                                   offsets are absolute addresses / elem size  */
  double* results;              /* 2 doubles per finaliser slot               */
  unsigned long long* timing;   /* optional: 2 per bucket (first start, last end, ns) */
  int64_t arena_elems;          /* arena size in elements (bounds checks of the
                                   QTN_DEBUG build; 0 = unchecked)             */
  /* n_in_elems: the arena's input region [0, n_in_elems) (gate tensors).
   * complex64 programs: inputs_hi holds the
   * same region as complex128 (the gates before narrowing) — K2 stages
   * compute in double precision and stage small input members from here in
   * shared memory before an item waits for its producers, so the
   * gates enter the contraction unrounded; only intermediates are stored as
   * complex64.  inputs_hi NULL (complex128 programs): no staging. */
  const void* inputs_hi;
  int64_t n_in_elems;
} qtn_program_t;

/* Execution node of a program graph.
 *  QTN_NODE_SMALL: a persistent launch over items [first, first + count) —
 *    the batched small-bucket schedule (K2): dependencies inside the stage
 *    are per-item completion counters, tickets are stage-relative.
 *  QTN_NODE_LARGE: one item, one launch of the large-item kernel (K1)
 *    specialised by `variant` (or K3 / K4 / K5 when the item has their
 *    shape) — or, count == 2, a producer / consumer PAIR: item `first`'s
 *    result is read by item first + 1 only, as a member carrying every
 *    result and summed index of the consumer.  The pair runs as ONE K6
 *    kernel (csrc/bucket_expand.cu: the producer's result never reaches
 *    HBM) when it has K6's shape, else as two kernels in sequence;
 *    n_tickets then holds the producer's K1 variant. */
enum { QTN_NODE_SMALL = 0, QTN_NODE_LARGE = 1 };
#define QTN_VARIANT_GENERIC (-1)
/* variant = log2(2^k) | (varying staged members) << 4 | (one streamed member) << 8
 *         | (varying members carrying result bit 0, complex64) << 12,
 * for k <= 3 and at most 4 varying members; otherwise QTN_VARIANT_GENERIC. */
typedef struct {
  int32_t kind;
  int32_t first;
  int32_t count;
  int32_t n_tickets;  /* SMALL: tickets of the stage                         */
  int32_t variant;    /* LARGE: kernel variant                               */
  int32_t dep_begin;  /* into the node dependency list                       */
  int32_t n_dep;
  int32_t smem_bytes; /* dynamic shared memory of the node's kernel          */
} qtn_node_t;

typedef struct qtn_graph qtn_graph_t;

/* ABI version (QTN_ABI_VERSION). */
int qtn_abi_version(void);
/* The routing / tuning knobs in effect ("name=value ..."): measured defaults,
 * overridden only by validated QTN_* environment variables read once per
 * process (csrc/knobs.h). */
const char* qtn_route_config(void);
/* Last error message of the calling thread ("" if none). */
const char* qtn_last_error(void);
/* Number of visible CUDA devices (0 on a CPU-only host; never fails). */
int qtn_device_count(int* count);
/* Zero the control block (ticket / exit counters and item completions). */
int qtn_program_reset(const qtn_program_t* prog, void* stream);
/* Launch one node (host-side description) on `stream`: the whole dependency
 * order of a program can be driven by issuing its nodes in a topological
 * order on one stream. */
int qtn_node_launch(const qtn_program_t* prog, const qtn_node_t* node, int32_t node_index, void* stream);
/* Build a CUDA graph of the program's nodes (node_deps holds, per node, the
 * indices of the nodes it waits for) on the current device. */
int qtn_graph_create(const qtn_program_t* prog, const qtn_node_t* nodes, int32_t n_nodes,
                     const int32_t* node_deps, qtn_graph_t** out);
/* Same, with the program's input upload (pinned host -> arena) as the graph's
 * first node and the result download (result slots -> pinned host) as its
 * last: one graph launch per contraction, end to end. */
typedef struct {
  const void* h2d_src;   /* pinned host input image                       */
  void* h2d_dst;         /* device arena (input region)                   */
  int64_t h2d_bytes;     /* 0 = no upload node                            */
  const void* d2h_src;   /* device result slots                           */
  void* d2h_dst;         /* pinned host result buffer                     */
  int64_t d2h_bytes;     /* 0 = no download node                          */
  /* Device-side input gather (instead of an upload node; n_gather > 0): a
   * first kernel node reads the RAW input tensors (complex128, concatenated
   * in pinned host memory, device-mapped) and writes input element t of the
   * canonical image: arena[gather_dst[t]] = narrowed raw[gather_src[t]] (and
   * inputs_hi[gather_dst[t]] = raw[gather_src[t]] for complex64 programs) —
   * no host-side gather, no copy-engine round trip. */
  const void* gather_raw;      /* pinned host, complex128                    */
  const int64_t* gather_src;   /* device: raw element per image element      */
  const int64_t* gather_dst;   /* device: arena element per image element     */
  int64_t n_gather;
} qtn_graph_io_t;
int qtn_graph_create_io(const qtn_program_t* prog, const qtn_node_t* nodes, int32_t n_nodes,
                        const int32_t* node_deps, const qtn_graph_io_t* io, qtn_graph_t** out);
/* Same, reading the item and member tables from HOST copies (the caller's
 * planner output, identical to what prog->buckets / prog->members hold on the
 * device) instead of copying them back: no synchronous device access, so a
 * graph can be built while earlier work still runs on the device.  io may be
 * NULL; host_members must hold every member the items reference. */
int qtn_graph_create_host(const qtn_program_t* prog, const qtn_bucket_t* host_items, const qtn_member_t* host_members,
                          int64_t n_host_members, const qtn_node_t* nodes, int32_t n_nodes,
                          const int32_t* node_deps, const qtn_graph_io_t* io, qtn_graph_t** out);
/* Launch the instantiated graph (one call per program execution). */
int qtn_graph_launch(qtn_graph_t* g, void* stream);
int qtn_graph_destroy(qtn_graph_t* g);
/* Kernel mix of a built graph: counts[6] = kernels of K1 (fused large-item
 * kernels), K2 (small-item stages), K3 (permutation-aware bucket kernel), K4
 * (expansion-item kernel), K5 (streaming-item kernel) and K6 (expansion item
 * fused with its consumer). */
int qtn_graph_kinds(const qtn_graph_t* g, int32_t* counts);
/* Per node (n = the graph's node count): 0 K1, 1 K2, 2 K3, 3 K4, 4 K5, 5 K6
 * (a pair node that fell back to two kernels reports its consumer's). */
int qtn_graph_node_kinds(const qtn_graph_t* g, int32_t* kinds, int32_t n);
/* Host planning (no device needed): the greedy min-fill (heuristic 0) or
 * min-degree (1) elimination order of a network given as CSR index lists
 * (tensor t holds tensor_idx[tensor_ptr[t] .. tensor_ptr[t+1])); open indices
 * are never eliminated.  Same heap discipline and smallest-id tie-breaks as
 * the reference's greedy_order (src/ordering.py:26-94), hence the same order.
 * order_out must hold every distinct index id; *n_out = entries written. */
int qtn_greedy_order(int32_t n_tensors, const int32_t* tensor_ptr, const int64_t* tensor_idx,
                     int32_t n_open, const int64_t* open_idx, int32_t heuristic,
                     int64_t* order_out, int32_t* n_out);
/* Host dry run (no device): the reference's symbolic bucket replay
 * (src/ordering.py:97-145) over CSR index lists with `fixed` (sliced) ids
 * removed: widths_out[i] = width of the bucket of active_out[i] (the order
 * without the fixed ids), *n_out = number of active ids.  widths_out and
 * active_out must hold n_order entries. */
int qtn_dry_run(int32_t n_tensors, const int32_t* tensor_ptr, const int64_t* tensor_idx, int32_t n_order,
                const int64_t* order, int32_t n_fixed, const int64_t* fixed, int32_t* widths_out,
                int64_t* active_out, int32_t* n_out);
/* Host greedy slicing (src/ordering.py:192-230): while the dry run is wider
 * than target_width, slice the smallest not-yet-sliced id of the widest
 * (first widest) bucket's union.  sliced_out holds up to max_out ids. */
int qtn_suggest_slicing(int32_t n_tensors, const int32_t* tensor_ptr, const int64_t* tensor_idx, int32_t n_order,
                        const int64_t* order, int32_t target_width, int32_t max_out, int64_t* sliced_out,
                        int32_t* n_out);
/* ---- Host program planner (no device needed) ----
 * qtn_plan_build replays the bucket assignment of the reference's
 * contract_network (src/ordering.py:165-187) over index sets only, merges
 * bucket chains into k-sum items under the engine's cost model and lays the
 * items out (tile bits, staging, step mask, member classes, kernel variant):
 * the C++ restatement of engine.plan_template (identical output, tested).
 * Input: CSR index lists in each tensor's own axis order, the elimination
 * order, the sliced (fixed) indices and the cost-model parameters.
 * Output arrays (int64, fetched by id after qtn_plan_array_len): */
enum {
  QTN_PLAN_W = 0, QTN_PLAN_K, QTN_PLAN_L, QTN_PLAN_LEVEL, QTN_PLAN_OUT_OFF, QTN_PLAN_MEM_PTR,
  QTN_PLAN_MEM_KIND, QTN_PLAN_MEM_REF, QTN_PLAN_MEM_MASK, QTN_PLAN_MEM_SMASK, QTN_PLAN_SMEM,
  QTN_PLAN_STMASK, QTN_PLAN_MEM_CLS, QTN_PLAN_VARIANT, QTN_PLAN_REF_W, QTN_PLAN_REF_ITEM,
  QTN_PLAN_REF_LAST, QTN_PLAN_REF_ELEMS, QTN_PLAN_BUCKET_INDEX, QTN_PLAN_FIN_KIND, QTN_PLAN_FIN_REF,
  QTN_PLAN_IN_OFF, QTN_PLAN_GDST, QTN_PLAN_GSRC, QTN_PLAN_GFIX, /* n_fixed rows of len(GDST) */
  QTN_PLAN_N_ARRAYS
};
typedef struct {
  int32_t elem_bytes, tile_bits, small_tile_bits, min_tile_bits;
  int32_t kmax, max_members, vec, nt;
  int32_t small_iter_bits, merge, resident_blocks;
  int64_t smem_budget;
  double hop_s, hop_k2_s, bw_bps, block_terms_ps, small_load_s;
  double cheap_member_w;  /* per-result weight of uniform / invariant members (1 = all equal) */
  int32_t kmax_large;     /* summed indices of a merged large (K1) item, <= 3            */
  int32_t wave_slots;     /* resident K1 blocks on the device (0 = no wave-aware tiles)   */
  int32_t wave_ov_elems;  /* per-tile fixed cost in result-element equivalents           */
} qtn_plan_params_t;
typedef struct qtn_plan qtn_plan_t;
int qtn_plan_build(int32_t n_tensors, const int32_t* tensor_ptr, const int64_t* tensor_idx,
                   int32_t n_order, const int64_t* order, int32_t n_fixed, const int64_t* fixed,
                   const qtn_plan_params_t* params, qtn_plan_t** out);
/* s[0] = input elements, s[1] = intermediate elements, s[2] = raw source
 * elements, s[3] = widest bucket. */
int qtn_plan_scalars(const qtn_plan_t* plan, int64_t* s);
int qtn_plan_array_len(const qtn_plan_t* plan, int32_t id, int64_t* len);
int qtn_plan_array(const qtn_plan_t* plan, int32_t id, int64_t* dst);
int qtn_plan_destroy(qtn_plan_t* plan);

/* dst[e] = convert(src[sum_j bit_j(e) * src_strides[j]]) for e < 2^rank,
 * j = 0 the fastest dst axis; src/dst element types given separately
 * (complex128 -> complex64 narrowing allowed).  General axis permutation +
 * slice offset for tensors entering a program in a non-canonical layout
 * (src/tensor_core.py:107-114, src/ordering.py:233-248). */
int qtn_permute(int32_t src_dtype, const void* src, int64_t src_offset,
                int32_t dst_dtype, void* dst, int32_t rank,
                const int64_t* src_strides, void* stream);

/* ---- K3: one standalone bucket, members in any axis order ----
 * The process-bucket call of the reference, contract_bucket(Bucket, Backend)
 * (src/tensor_core.py:167-188) with the fast_kernel body
 * (src/tensor_core.py:148-164), for members that are NOT in the program's
 * canonical layout (arbitrary index permutations, strided slices): no member
 * is transposed in HBM first.  Iteration bit b < w is result axis b of the
 * sorted result (b = 0 the LAST sorted index, i.e. the fastest axis of the C
 * order output, src/tensor_core.py:117-122); bit w is the bucket index.
 *     out[r] = sum_{s=0,1} prod_i data_i[sum_b bit_b(r, s) * strides_i[b]]
 * members multiplied in order, s = 0 then s = 1.  Every member must carry
 * the bucket index (strides[w] > 0, reference: Bucket validation,
 * src/tensor_core.py:86-90); w <= 31, member rank <= 32. */
typedef struct {
  const void* data;                   /* device pointer (element aligned)           */
  int64_t strides[QTN_MAX_WIDTH + 1]; /* element stride per iteration bit, 0 = absent */
} qtn_bmember_t;

typedef struct {
  int32_t dtype;   /* QTN_C64 / QTN_C128 (members and output)                   */
  int32_t w;       /* result rank                                               */
  int32_t n_mem;   /* 1..QTN_MAX_MEMBERS                                        */
  int32_t k;       /* summed indices, iteration bits w .. w+k-1 (0 or 1: one
                      bucket index; up to 3: a merged chain of buckets — the
                      members then need not carry every summed index)       */
  void* out;       /* 2^w elements, C order over the sorted result indices      */
  qtn_bmember_t mem[QTN_MAX_MEMBERS];
} qtn_bucket_desc_t;

/* Launch K3 on `stream` (asynchronous; buffers must stay alive until the
 * stream is synchronised).  Errors: QTN_E_INVALID (bad descriptor),
 * QTN_E_UNSUPPORTED (w > 31, rank > 32), QTN_E_CUDA. */
int qtn_bucket(const qtn_bucket_desc_t* desc, void* stream);
/* out[r] = sum over the 2^k assignments s of the summed bits (ascending) of
 * prod_i data_i[...]; k > 1 is the program path's merged-chain form. */
/* Plan only (no device), info[8]: [0] tile bits, [1] staged elements per
 * tile, [2] shared-memory bytes per block, [3] tiles, [4] staged members
 * (-1 = every member staged, generic kernel), [5] members folded into the
 * per-tile product table, [6] product-table bits. */
int qtn_bucket_plan(const qtn_bucket_desc_t* desc, int32_t* info);

/* ---- K4: an expansion bucket (one dominant member) ----
 * Same contraction as qtn_bucket for a descriptor whose dominant member (the
 * one with the most result bits) lacks between min_e (>= 0) and 8 result bits
 * ("expansion bits"), k in 1..3, 8 <= w <= 31, the other members' bits inside
 * the K4 tile <= 12 (c64) / 11 (c128) with the summed bits.  The dominant
 * member is read once into registers, the others through a per-tile product
 * table (csrc/bucket_expand.cu).  Program graphs route their expansion items
 * here (QTN_K4).  QTN_E_UNSUPPORTED when the bucket is not such an expansion. */
int qtn_bucket_expand(const qtn_bucket_desc_t* desc, int32_t min_e, void* stream);

/* ---- K5: a streaming bucket (one member carries every result bit) ----
 * Same contraction for a descriptor in which one member carries all w
 * result bits (k in 1..3, at most 4 members carry result bits, w >= 8 / 9 at
 * complex128 / complex64): that member is streamed once, the others read
 * directly through L1/L2 (csrc/bucket_stream.cu).  Program graphs route
 * their streaming items here (QTN_K5).  QTN_E_UNSUPPORTED otherwise. */
int qtn_bucket_stream(const qtn_bucket_desc_t* desc, void* stream);

/* ---- K6: an expansion bucket fused with its only consumer ----
 * `producer` is a K4-shaped bucket (qtn_bucket_expand) whose result is member
 * `member` of `consumer`, carrying every result and summed index of the
 * consumer in order (consumer->mem[member].data == producer->out, strides
 * 1, 2, 4, ... over the consumer's w + k iteration bits; producer->w ==
 * consumer->w + consumer->k, consumer k in 1..3).  Computes the consumer's
 * result without materialising the producer's: producer->out is NOT written
 * (it may be any non-null pointer).  Same sum order as the two buckets run
 * one after the other; the intermediate is not rounded to the element type.
 * QTN_E_UNSUPPORTED when the pair does not have that shape. */
int qtn_bucket_expand_fused(const qtn_bucket_desc_t* producer, const qtn_bucket_desc_t* consumer,
                            int32_t member, void* stream);
/* Plan only (no device): info[8] = producer summed bits, consumer summed
 * bits, expansion bits, product-table bits, gathered consumer members,
 * uniform consumer members, consumer summed bits no gathered member carries,
 * tile-id bits.  Same errors as qtn_bucket_expand_fused. */
int qtn_bucket_expand_fused_plan(const qtn_bucket_desc_t* producer, const qtn_bucket_desc_t* consumer,
                                 int32_t member, int32_t* info);

#ifdef __cplusplus
}
#endif
#endif /* QTN_B200_H */
