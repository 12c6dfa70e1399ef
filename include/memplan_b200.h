/* memplan_b200 — B200-native (sm_100a) data-parallel core of the OLLA memory
 * planner (arXiv 2210.12924), behind a plain C ABI.
 *
 * This header is the drop-in boundary. Every entry point names the
 * reference interface it replaces (file:line under /root/reference/proj).
 * The reference has no FFI of its own (it is a static C++ library,
 * CMakeLists.txt:10-25); INTEGRATION.md shows the C++ shim a maintainer adds
 * so memplan's pipeline/CLI call these functions with their existing
 * signatures, and the ctypes binding the Python tests use.
 *
 * Conventions
 *   - Indices are int32 (memplan::NodeIndex / EdgeIndex are `int`,
 *     graph.hpp:58-59); byte sizes and addresses are uint64.
 *   - Timesteps are 1-based and intervals closed, as memplan::Interval
 *     (analysis.hpp:28-37); an interval with lo > hi is empty.
 *   - Functions without the `_d` suffix take HOST buffers and copy in/out on
 *     the context's stream (mp_ctx_set_stream) and return when done.
 *     `_d` variants take DEVICE pointers and a cudaStream_t (as void*; NULL
 *     is the default stream, as in every CUDA API), are stream-ordered and
 *     never synchronise unless stated (the pair/validation counts do).
 *   - No CPU fallback exists: with no usable sm_100 device every call that
 *     computes returns MP_E_NO_DEVICE / MP_E_CUDA.
 *   - Errors map 1:1 onto the reference's exception classes
 *     (errors.hpp:24-76); mp_last_error() returns the reference-format
 *     message ("InvalidOrder: sequence is not a topological order of the
 *     graph", schedule.cpp:25-26).
 */
#ifndef MEMPLAN_B200_H_
#define MEMPLAN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MP_ABI_VERSION 1

typedef enum {
  MP_OK = 0,
  MP_E_INVALID_ORDER = 1, /* memplan::InvalidOrder (schedule.cpp:25, plan.cpp:107) */
  MP_E_BAD_GRAPH = 2,     /* DanglingEndpoint / InvalidStructure analogues (graph.cpp:64-141) */
  MP_E_INVALID_ARG = 3,   /* null pointer, negative size, mismatched lengths */
  MP_E_CUDA = 4,          /* CUDA runtime failure (message in mp_last_error) */
  MP_E_OOM = 5,           /* device allocation failed */
  MP_E_CAPACITY = 6,      /* caller buffer smaller than the result (count returned) */
  MP_E_NO_DEVICE = 7      /* no sm_100 device: there is no CPU fallback */
} mp_status;

typedef struct mp_ctx mp_ctx;     /* one device + one stream + scratch */
typedef struct mp_graph mp_graph; /* device-resident graph (CSR + derived tables) */

/* Flattened memplan::Graph (graph.hpp:62-127): edge e is produced by
 * edge_src[e] and consumed by sinks[sink_off[e] .. sink_off[e+1]).
 * edge_size[e] == 0 marks a control edge (graph.cpp:89-93): it orders nodes
 * but carries no bytes. Node order is program order. */
typedef struct {
  int32_t num_nodes;
  int32_t num_edges;
  const int32_t* edge_src;   /* [num_edges] */
  const int64_t* sink_off;   /* [num_edges + 1] */
  const int32_t* sinks;      /* [sink_off[num_edges]] */
  const uint64_t* edge_size; /* [num_edges] */
} mp_csr;

typedef struct {
  int32_t num_nodes;
  int32_t num_edges;
  int64_t num_sinks;
  int64_t num_pred_pairs;  /* distinct (producer, consumer) node pairs checked for validity */
  int32_t num_multi_sink;  /* data edges whose last consumer depends on the order */
  int32_t smem_resident;   /* 1 when the fused scorer keeps per-candidate state in smem */
  uint64_t total_bytes;    /* Graph::total_bytes() (graph.hpp:93) */
  int32_t orders16;        /* host-buffer scoring's wire format: 1 uint16 ids (half the bytes),
                              2 3-byte ids (three quarters), 0 int32 */
  int32_t score_variant;   /* MP_SCORER_*: which fused-scorer formulation the graph got */
} mp_graph_info;
#define MP_SCORER_REG 1      /* register slots, per-candidate state in smem (n up to ~8k) */
#define MP_SCORER_SMEM 2     /* node tables from global, state in smem (n < 65536) */
#define MP_SCORER_WARP 3     /* warp per candidate (opt-in, n <= 2048) */
#define MP_SCORER_SCRATCH 4  /* per-CTA global position scratch (large graphs) */
#define MP_SCORER_PARTS 5    /* node-partitioned passes, positions in smem (large graphs) */

/* ---- context / graph lifetime --------------------------------------------- */
int mp_abi_version(void);
const char* mp_status_string(mp_status s);
const char* mp_last_error(void); /* thread-local, reference-format message */

mp_status mp_ctx_create(int device, mp_ctx** out);
mp_status mp_ctx_destroy(mp_ctx* ctx);
/* Use a caller stream (cudaStream_t as void*) instead of the context's own. */
mp_status mp_ctx_set_stream(mp_ctx* ctx, void* stream);
mp_status mp_ctx_synchronize(mp_ctx* ctx);

/* Validates and uploads a graph once (the analogue of Graph::build,
 * graph.cpp:64-141, for the checks the kernels rely on: endpoints in range,
 * monotone sink offsets, no duplicate sink within one edge). */
mp_status mp_graph_upload(mp_ctx* ctx, const mp_csr* csr, mp_graph** out);
mp_status mp_graph_free(mp_graph* g);
mp_status mp_graph_get_info(const mp_graph* g, mp_graph_info* info);

/* Host-only diagnostic of the node partition the large-graph scorer would use
 * (MP_SCORER_PARTS): info[7] = {parts, max local slots per part,
 * stash slots, cross-part validity pairs, cross-part multi-consumer tensors,
 * shared-memory bytes, tiny4}; parts = 0 when no partition fits smem_budget. */
mp_status mp_parts_plan_host(const mp_csr* csr, int32_t max_chunks, int64_t smem_budget,
                             int64_t* info);

/* Host-only (no device): the scorer's derived validity and free tables for a
 * graph (mp_prep.cpp, run by mp_graph_upload). info[7] = {reduced validity pairs,
 * multi-consumer (order-dependent free) tensors, exact reachability (1) or the
 * chain index (0), tiny4, tiny8, narrow (32-bit sums), mid32 (32-bit per-node
 * values, 64-bit sums)}. When pairs != NULL it
 * receives up to `cap` reduced pairs as (u, w) int32 couples: u must run before w. */
mp_status mp_prep_host(const mp_csr* csr, int64_t* info, int32_t* pairs, int64_t cap);

/* ---- (a2/a3) lifetimes over one order ---------------------------------------
 * memplan::lifetimes_from_order (schedule.cpp:33-50) incl. the
 * is_topological_order verdict (graph.cpp:239-254): returns
 * MP_E_INVALID_ORDER for a non-topological order. lo/hi: [num_edges]. */
mp_status mp_lifetimes(mp_ctx* ctx, const mp_graph* g, const int32_t* order, int64_t order_len,
                       int32_t* lo, int32_t* hi);
mp_status mp_lifetimes_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_order,
                         int64_t order_len, int32_t* d_lo, int32_t* d_hi, int32_t* d_valid,
                         void* stream);

/* ---- (a4) realized lifetimes -------------------------------------------------
 * memplan::realized_lifetimes (plan.cpp:101-120). timestep_of[v] == 0 means
 * node v has no timestep; the first such node met in edge order (source,
 * then sinks) yields MP_E_INVALID_ORDER "node <id> has no timestep" — the
 * node index is returned in *missing_node (ids live on the host side). */
mp_status mp_realized_lifetimes(mp_ctx* ctx, const mp_graph* g, const int32_t* timestep_of,
                                int32_t horizon, int32_t* lo, int32_t* hi,
                                int32_t* missing_node);

/* ---- (a8/a9/a10) resident bytes ---------------------------------------------
 * resident_bytes_per_step / peak_resident_bytes (schedule.cpp:69-88). */
mp_status mp_resident_bytes(mp_ctx* ctx, const mp_graph* g, const int32_t* order,
                            int64_t order_len, uint64_t* bytes /* [num_nodes] */);
mp_status mp_peak_resident_bytes(mp_ctx* ctx, const mp_graph* g, const int32_t* order,
                                 int64_t order_len, uint64_t* peak);
/* timeline_from_lifetimes (plan.cpp:122-143): bytes per step over
 * 1..horizon (bytes may be NULL), peak_rs and peak_step (first strict
 * maximum; 1 when all zero and horizon > 0; 0 when horizon == 0). */
mp_status mp_timeline(mp_ctx* ctx, const mp_graph* g, const int32_t* lo, const int32_t* hi,
                      int32_t horizon, uint64_t* bytes, uint64_t* peak_rs, int32_t* peak_step);

/* ---- batched candidate scoring (K1+K3 fused) ----------------------------------
 * For each candidate order c (row c of [num_orders][num_nodes] int32):
 * valid[c] = is_topological_order (graph.cpp:239-254); when valid,
 * peak[c] = peak_resident_bytes (schedule.cpp:81-88) and peak_step[c] the
 * first step attaining it (plan.cpp:135-141); invalid candidates get
 * peak = 0, peak_step = 0. The multi-order analogue of
 * enumerate_min_peak's scoring (oracle.cpp:74-93). */
mp_status mp_score_orders(mp_ctx* ctx, const mp_graph* g, const int32_t* orders,
                          int64_t num_orders, uint64_t* peak, int32_t* peak_step,
                          uint8_t* valid);
mp_status mp_score_orders_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_orders,
                            int64_t num_orders, uint64_t* d_peak, int32_t* d_peak_step,
                            uint8_t* d_valid, void* stream);
/* Scoring with the argmin fused in: *best = first-minimum index over valid
 * candidates (-1 if none). One kernel on the device; host buffers. */
mp_status mp_score_orders_best(mp_ctx* ctx, const mp_graph* g, const int32_t* orders,
                               int64_t num_orders, uint64_t* peak, int32_t* peak_step,
                               uint8_t* valid, int64_t* best);
/* Device variant of the fused form. d_best_key points to TWO words
 * {key, overflow}, reset to {MP_KEY_NONE, MP_KEY_NONE} by one byte memset
 * (mp_key_reset_d, stream-ordered; a memset node inside a CUDA graph). Every
 * valid candidate c with peak < 2^42 and c + index_base < 2^20 does
 * atomicMin(&key, peak << 20 | (c + index_base)); any other valid candidate
 * sets overflow = 0, telling the caller to fall back to mp_argmin_key_d.
 * Both words are non-negative int64 values, so one int64 allreduce(MIN) of
 * the pair across GPUs yields the global first-minimum AND whether any shard
 * overflowed. */
#define MP_KEY_NONE 0x7f7f7f7f7f7f7f7full
#define MP_KEY_OVERFLOW 0x7f7f7f7f7f7f7f7eull /* mp_argmin_key_d d_out3[2] only */
#define MP_KEY_MAX_PEAK (1ull << 42)
mp_status mp_key_reset_d(mp_ctx* ctx, uint64_t* d_best_key, void* stream);
mp_status mp_score_orders_argmin_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_orders,
                                   int64_t num_orders, uint64_t* d_peak, int32_t* d_peak_step,
                                   uint8_t* d_valid, uint64_t* d_best_key, int64_t index_base,
                                   void* stream);
/* First-minimum argmin over valid candidates (oracle.cpp:78-81 keeps the
 * first strictly smaller peak): *best = index or -1 when none is valid. */
mp_status mp_argmin(mp_ctx* ctx, const uint64_t* peak, const uint8_t* valid, int64_t num_orders,
                    int64_t* best);
/* Device variant (one CTA): d_out3[0] = best index + index_base (or -1),
 * d_out3[1] = its peak, d_out3[2] = packed key peak << 20 | index
 * (MP_KEY_NONE when nothing is valid, MP_KEY_OVERFLOW when peak >= 2^42 or
 * index >= 2^20). index_base makes keys of different GPU shards comparable. */
mp_status mp_argmin_key_d(mp_ctx* ctx, const uint64_t* d_peak, const uint8_t* d_valid,
                          int64_t num_orders, int64_t index_base, uint64_t* d_out3,
                          void* stream);

/* ---- (a6) liveness-overlap pairs --------------------------------------------
 * The pair set of encode_addresses' loop (encode.cpp:347-367): i < j in
 * edge-index order, size[i] > 0 and size[j] > 0 (encode.cpp:329-331), not
 * both pinned (:351), closed intervals intersecting (:354). The
 * edge_precedes filter (:355-357) removes nothing on lifetimes realized from
 * a topological order, which is the contract here.
 * pinned may be NULL. Two-phase: call with pairs == NULL for the count;
 * pairs is [cap][2] int32 in lexicographic (i, j) order. */
mp_status mp_overlap_pairs(mp_ctx* ctx, int32_t num_edges, const int32_t* lo, const int32_t* hi,
                           const uint64_t* size, const uint8_t* pinned, int32_t* pairs,
                           int64_t cap, int64_t* count);
/* Device variant over a row range [row_begin, row_end) (for sharding rows
 * across GPUs): d_row_off[row_end-row_begin+1] (int64) receives the
 * exclusive offsets (relative to the range). With d_pairs != NULL the count,
 * scan and fill run back to back on the stream (one read-back of the total at
 * the end): at most cap pairs are written, MP_E_CAPACITY when the total exceeds
 * cap (*count still receives the total). */
mp_status mp_overlap_pairs_d(mp_ctx* ctx, int32_t num_edges, const int32_t* d_lo,
                             const int32_t* d_hi, const uint64_t* d_size,
                             const uint8_t* d_pinned, int64_t row_begin, int64_t row_end,
                             int64_t* d_row_off, int32_t* d_pairs, int64_t cap,
                             int64_t* count, void* stream);

/* ---- (a11/a12/a13) address-plan validation + fragmentation ---------------------
 * Pairwise part of validate_plan (plan.cpp:390-404): among edges with
 * size > 0 and has_addr != 0, pairs i < j whose closed lifetimes intersect
 * and whose [addr, addr+size) ranges overlap. Violating pairs come back in
 * (i, j) order (viol [cap][2], may be NULL for the count). */
mp_status mp_validate_pairs(mp_ctx* ctx, int32_t num_edges, const int32_t* lo, const int32_t* hi,
                            const uint64_t* size, const uint8_t* has_addr, const uint64_t* addr,
                            int32_t* viol, int64_t cap, int64_t* num_viol);
mp_status mp_validate_pairs_d(mp_ctx* ctx, int32_t num_edges, const int32_t* d_lo,
                              const int32_t* d_hi, const uint64_t* d_size,
                              const uint8_t* d_has_addr, const uint64_t* d_addr,
                              int64_t row_begin, int64_t row_end, int64_t* d_row_off,
                              int32_t* d_viol, int64_t cap, int64_t* num_viol, void* stream);
/* addresses_feasible (pipeline.cpp:146-160): *feasible = 1 iff no
 * conflicting pair among edges with has_addr. */
mp_status mp_addresses_feasible(mp_ctx* ctx, int32_t num_edges, const int32_t* lo,
                                const int32_t* hi, const uint64_t* size,
                                const uint8_t* has_addr, const uint64_t* addr, int32_t* feasible);
/* peak_mem = max(addr + size) over edges with an address (pipeline.cpp:270-275). */
mp_status mp_peak_mem(mp_ctx* ctx, int32_t num_edges, const uint64_t* size,
                      const uint8_t* has_addr, const uint64_t* addr, uint64_t* peak_mem);
/* fragmentation (placement.cpp:64-67): (mr - rs) / mr, 0 when mr == 0. */
double mp_fragmentation(uint64_t mr, uint64_t rs);

/* ---- (e) one process, several GPUs --------------------------------------------
 * A set of contexts (one per entry of devices[G]; an entry may repeat) with the
 * graph replicated on each (the CSR is replicated, candidates
 * sharded). mp_score_orders_multi splits orders [num_orders][n] into G
 * contiguous shards, scores each on its device from its own host thread (the
 * fused kernel with its argmin), and combines the per-device first minima on
 * the host: *best is the lowest index among equal minimal peaks over all
 * shards, exactly a serial first-minimum scan (-1 when nothing is valid).
 * With distinct devices and NCCL present (loaded at run time), mp_multi_create
 * makes one communicator per device (ncclCommInitAll) and the shards' fused
 * {key, overflow} pairs meet in ONE device-side ncclAllReduce(MIN);
 * the host combine remains only for repeated devices, a missing NCCL, or a key
 * that does not fit (mp_multi_nccl tells which path is active).
 * Multi-process jobs use the same kernels with one NCCL allreduce(MIN) on the
 * packed key instead (mp_score_orders_argmin_d + paper_2210_12924_b200/dist.py). */
typedef struct mp_multi mp_multi;
mp_status mp_multi_create(const int* devices, int num_devices, mp_multi** out);
mp_status mp_multi_destroy(mp_multi* m);
mp_status mp_multi_upload(mp_multi* m, const mp_csr* csr);
int mp_multi_nccl(const mp_multi* m);
mp_status mp_score_orders_multi(mp_multi* m, const int32_t* orders, int64_t num_orders,
                                uint64_t* peak, int32_t* peak_step, uint8_t* valid,
                                int64_t* best);

/* ---- (§8f-2) placement heuristics: the producers of the plans K4 validates ----
 * preallocate_pyramid (placement.cpp:25-62) and greedy_pack
 * (placement.cpp:182-204) over num_problems lifetime vectors that share the
 * edge sizes (problem b: lo/hi [b*num_edges ..], e.g. one per candidate order),
 * plus peak_mem = max(addr + size) of the result (pipeline.cpp:270-275).
 * flags: MP_PLACE_PYRAMID      the preplaced map is preallocate_pyramid's
 *                              (pipeline.cpp:248-249); fixed must be NULL
 *        MP_PLACE_PYRAMID_ONLY stop after the pyramid (PrePlacement.assigned)
 * fixed / fixed_addr [num_edges]: the caller's preplaced map (may be NULL).
 * id_rank [num_edges]: rank of each edge id in byte-lexicographic order, the
 * pyramid's last tie-break (placement.cpp:48-50); NULL = edge index order.
 * Outputs: addr / has_addr [num_problems][num_edges] (has_addr = the edge is in
 * the returned map), peak_mem [num_problems] and pyramid_base
 * [num_problems] (PrePlacement.reserved_base), both optional.
 * Up to 8192 edges per problem the placed set lives in shared memory (many
 * problems per SM); larger graphs (up to 2^18 - 1 edges, e.g. the 100k-tensor
 * graph) keep it in a per-CTA global slice, one problem per SM. Past that:
 * MP_E_CAPACITY. */
#define MP_PLACE_PYRAMID 1u
#define MP_PLACE_PYRAMID_ONLY 2u
mp_status mp_place(mp_ctx* ctx, int32_t num_edges, int64_t num_problems, const int32_t* lo,
                   const int32_t* hi, const uint64_t* size, const int32_t* id_rank,
                   const uint8_t* fixed, const uint64_t* fixed_addr, uint32_t flags,
                   uint64_t* addr, uint8_t* has_addr, uint64_t* peak_mem,
                   uint64_t* pyramid_base);
mp_status mp_place_d(mp_ctx* ctx, int32_t num_edges, int64_t num_problems, const int32_t* d_lo,
                     const int32_t* d_hi, const uint64_t* d_size, const int32_t* d_id_rank,
                     const uint8_t* d_fixed, const uint64_t* d_fixed_addr, uint32_t flags,
                     uint64_t* d_addr, uint8_t* d_has_addr, uint64_t* d_peak_mem,
                     uint64_t* d_pyramid_base, void* stream);

/* ---- batched candidate PLANS: plan_once's placement half per candidate order ----
 * For each candidate order c (row c of [num_orders][num_nodes]):
 *   schedule score  valid[c], peak_rs[c], peak_step[c] as mp_score_orders;
 *   lifetimes_from_order (schedule.cpp:33-50) of the order;
 *   addresses       preallocate_pyramid (flags & MP_PLACE_PYRAMID) then greedy_pack
 *                   (placement.cpp:25-62, 182-204) over those lifetimes, as plan_once's
 *                   preplacement + greedy placement (pipeline.cpp:101-109, 248-249);
 *   peak_mem[c]     max(addr + size) (pipeline.cpp:270-275);
 *   nviol[c]        the address check: pairs validate_plan reports as below_above
 *                   (plan.cpp:390-404; addresses_feasible, pipeline.cpp:146-160, is
 *                   nviol == 0). Invalid orders get nviol = 0, peak_mem = 0.
 * d_addr / d_has_addr [num_orders][num_edges] may be NULL (context scratch).
 * d_best_key (optional, 2 words as mp_score_orders_argmin_d): first minimum of
 * peak_mem over feasible plans (valid order, nviol == 0). Stream-ordered; the
 * placement bounds apply (num_edges <= 2^18 - 1). Past the shared-memory kernels
 * (8192 edges, or positions / pair records beyond shared memory) the lifetimes run
 * per candidate, the placement one problem per SM, the check as a K4 sweep per plan. */
mp_status mp_score_plans_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_orders,
                           int64_t num_orders, const int32_t* d_id_rank, uint32_t flags,
                           uint64_t* d_peak_rs, int32_t* d_peak_step, uint8_t* d_valid,
                           uint64_t* d_peak_mem, uint32_t* d_nviol, uint64_t* d_addr,
                           uint8_t* d_has_addr, uint64_t* d_best_key, int64_t index_base,
                           void* stream);
/* The address check alone, for caller-supplied plans: per plan c the number of
 * pairs validate_plan reports as below_above (plan.cpp:390-404) given the plan's
 * lifetimes lo/hi and addresses addr/has_addr ([num_plans][num_edges] each; size
 * [num_edges] shared). Plans with valid[c] == 0 (optional) are skipped (nviol 0,
 * peak_mem untouched when d_peak_mem is NULL). num_edges <= 8192. */
mp_status mp_validate_plans_d(mp_ctx* ctx, int32_t num_edges, int64_t num_plans,
                              const int32_t* d_lo, const int32_t* d_hi, const uint64_t* d_size,
                              const uint8_t* d_has_addr, const uint64_t* d_addr,
                              const uint8_t* d_valid, uint32_t* d_nviol, void* stream);
/* lifetimes_from_order for many orders at once (schedule.cpp:33-50): lo/hi
 * [num_orders][num_edges] int32 (1-based), valid[c] = is_topological_order. */
mp_status mp_lifetimes_batch_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_orders,
                               int64_t num_orders, int32_t* d_lo, int32_t* d_hi,
                               uint8_t* d_valid, void* stream);

/* ---- (§8f-1) non-overlap rows: the external-ILP model text from the GPU pair list ----
 * write_lp(encode_addresses(graph, lifetimes, preplaced)) (lp_format.cpp:88-121,
 * encode.cpp:320-377) as text: per overlapping pair (the K2 pair set, i.e.
 * filter_pairs on realized lifetimes) the live_pair / below /
 * above rows and its two binaries, formatted on the GPU; the O(num_edges)
 * sections (objective, peak_address rows, Bounds, Generals) on the host.
 * ids: the edge ids concatenated, id_off [num_edges + 1] byte offsets (the
 * variable names, sanitized as lp_format.cpp:30-36). pinned / pinned_addr: the
 * preplaced map (may be NULL). Two-phase: out == NULL returns *len only.
 * counts [4] (optional): rows tagged live_pair, below, above, peak_address.
 * Ids that sanitize ambiguously (where lp_names would append "_2") are
 * refused with MP_E_INVALID_ARG. */
mp_status mp_encode_addresses_lp(mp_ctx* ctx, int32_t num_edges, const int32_t* lo,
                                 const int32_t* hi, const uint64_t* size, const uint8_t* pinned,
                                 const uint64_t* pinned_addr, const char* ids,
                                 const int64_t* id_off, char* out, int64_t cap, int64_t* len,
                                 int64_t* counts);

/* ---- (§8f-3) joint-mode pair set ------------------------------------------------
 * The pair loop of encode_joint (encode.cpp:401-408): data edges i < j, minus
 * those ordered by the graph (edge_precedes either way, analysis.cpp:94-113,
 * with compute_bounds' windows, analysis.cpp:33-62) when filter != 0. Pairs
 * come back in the reference's (i, j) order; two-phase (pairs == NULL: count).
 * Graphs over 32,768 nodes return MP_E_CAPACITY (host descendant bitsets). */
mp_status mp_joint_pairs(mp_ctx* ctx, const mp_graph* g, int filter, int32_t* pairs, int64_t cap,
                         int64_t* count);

/* ---- (§8f-4) arena baseline: run_baseline over candidate orders ---------------
 * run_baseline (placement.cpp:150-180): the free-list Arena (placement.cpp:69-148,
 * first fit, or best fit when best_fit != 0) replayed over every order of
 * orders [num_orders][n]: mr_peak (allocator high-water mark), rs_at_peak (live
 * bytes when it was set) and fragmentation (placement.cpp:64-67, computed in
 * double as the reference does). valid[c] = 0 where the reference throws
 * InvalidOrder (the other outputs are then 0). Returns MP_E_CAPACITY when the
 * per-candidate state (about 4 n + 20 num_edges bytes) exceeds shared memory. */
mp_status mp_run_baseline(mp_ctx* ctx, const mp_graph* g, const int32_t* orders,
                          int64_t num_orders, int best_fit, uint64_t* mr_peak,
                          uint64_t* rs_at_peak, double* fragmentation, uint8_t* valid);
mp_status mp_run_baseline_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_orders,
                            int64_t num_orders, int best_fit, uint64_t* d_mr_peak,
                            uint64_t* d_rs_at_peak, double* d_fragmentation, uint8_t* d_valid,
                            void* stream);

/* ---- workload helpers (host C++, not on the measured path) ----------------------
 * Deterministic graph families with the semantics of generate_graph
 * (generate.cpp:45-158; chain = 0, fork_join = 1, training_like = 2).
 * Two-phase: call with NULL arrays to get the dims. Node/edge ids are not
 * produced (the CSR is id-free); training_like's naming is documented in
 * paper_2210_12924_b200/graph.py. */
mp_status mp_generate_graph(int kind, int32_t layers, uint64_t size, uint64_t seed,
                            int32_t* num_nodes, int32_t* num_edges, int64_t* num_sinks,
                            int32_t* edge_src, int64_t* sink_off, int32_t* sinks,
                            uint64_t* edge_size, uint8_t* node_role);
/* Seeded uniformly-random topological orders (randomised Kahn; candidate c
 * uses a splitmix64 stream seeded from (seed, c)). out: [num_orders][n]. */
mp_status mp_random_topo_orders(const mp_csr* csr, int64_t num_orders, uint64_t seed,
                                int32_t num_threads, int32_t* out);

#ifdef __cplusplus
}
#endif

#endif /* MEMPLAN_B200_H_ */
