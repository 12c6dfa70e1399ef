// Internal types shared by the memplan_b200 CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "memplan_b200.h"

namespace mpb {

// Thread-local error text behind mp_last_error().
void set_error(const std::string& msg);

// Returns MP_E_CUDA / MP_E_OOM with a message when `e` is an error.
mp_status cuda_status(cudaError_t e, const char* what);

#define MP_CUDA(expr)                                             \
  do {                                                            \
    cudaError_t _e = (expr);                                      \
    if (_e != cudaSuccess) return ::mpb::cuda_status(_e, #expr);  \
  } while (0)

#define MP_TRY(expr)                    \
  do {                                  \
    mp_status _s = (expr);              \
    if (_s != MP_OK) return _s;         \
  } while (0)

// Growable device scratch owned by a context (never shrinks).
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
  mp_status reserve(size_t want);
  ~Scratch();
};

}  // namespace mpb

struct mp_ctx {
  int device = 0;
  int num_sms = 0;
  size_t max_smem_optin = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;  // own_stream unless mp_ctx_set_stream
  mpb::Scratch scratch[8];        // independent scratch slots per call site
  mpb::Scratch host_pinned_dummy;
  // small device buffer for per-call flags / counters
  int64_t* d_small = nullptr;
  // host-buffer scoring pipeline: a copy stream, per-chunk events, a pinned word pair
  cudaStream_t copy_stream = nullptr;
  static constexpr int kPipeChunks = 8;
  cudaEvent_t ev_h2d[kPipeChunks] = {};
  cudaEvent_t ev_start = nullptr;
  uint64_t* h_small = nullptr;  // pinned: [0] key init, [1] key read-back
  uint8_t* h_stage = nullptr;   // pinned: two halves of packed (16/24-bit) orders
  size_t h_stage_bytes = 0;     // per half
  char* h_bounce = nullptr;     // pinned: two halves for large results to pageable memory
  cudaEvent_t ev_d2h[2] = {};
};

// Several contexts in one process, the graph replicated on each (mp_score_orders_multi).
// With distinct devices and libnccl available, one NCCL communicator per device
// (ncclCommInitAll) reduces the fused argmin key on the devices.
struct mp_multi {
  std::vector<mp_ctx*> ctx;
  std::vector<mp_graph*> graph;
  std::vector<void*> comm;  // ncclComm_t per context, empty without NCCL
  std::string nccl_note;    // why NCCL is not used (empty when it is)
};

// Device-resident graph tables. Built once by mp_graph_upload from the
// reference-shaped CSR (memplan::Graph flattened).
//
// Scoring tables (see mp_prep.cpp and DESIGN.md §3): reduced validity
// edges, per-node allocated / statically freed bytes, and the data edges
// whose last consumer depends on the order.
struct mp_graph {
  mp_ctx* ctx = nullptr;
  int32_t n = 0;
  int32_t E = 0;
  int64_t S = 0;
  uint64_t total_bytes = 0;

  // raw CSR (edge space)
  int32_t* d_edge_src = nullptr;
  int64_t* d_sink_off = nullptr;
  int32_t* d_sinks = nullptr;
  uint64_t* d_edge_size = nullptr;
  uint32_t* d_edge_size32 = nullptr;  // size / scale when `narrow` (the arena's 32-bit blocks)

  // node space, derived by mp_prep.cpp (scaled by `scale`)
  int64_t n_preds = 0;               // reduced validity edges (first + extra)
  int32_t n_extra = 0;               // reduced pairs beyond each node's first producer
  int32_t n_dyn = 0;                 // data edges whose last consumer depends on the order
  int32_t n_dyn_sinks = 0;
  int32_t dyn_max_sinks = 0;         // most candidate last consumers of one dynamic edge
  uint64_t scale = 1;
  bool narrow = true;
  bool mid32 = false;                // 32-bit scan inputs, 64-bit sums (mp_prep.h)
  bool tiny8 = false;                // per-position (x, f) fit a byte each (mp_prep.h)
  bool tiny4 = false;                // ... fit 4 bits each
  bool exact_reach = false;
  uint64_t* d_node_x = nullptr;      // [n] alloc - static free (scaled, modular)
  uint64_t* d_node_f = nullptr;      // [n] static free (scaled)
  int32_t* d_pred1 = nullptr;        // [n] first reduced producer or -1
  int32_t* d_extra_u = nullptr;      // [n_extra]
  int32_t* d_extra_w = nullptr;      // [n_extra]
  int32_t* d_dyn_off = nullptr;      // [n_dyn+1]
  int32_t* d_dyn_sinks = nullptr;    // [n_dyn_sinks]
  int32_t* d_dyn_sink4 = nullptr;    // [4 n_dyn] when every dynamic edge has <= 4 candidates
  uint64_t* d_dyn_size = nullptr;    // [n_dyn] scaled
  uint32_t* d_node_rec32 = nullptr;    // [4n] (x, f, pred1, pred2), 32-bit graphs
  int32_t* d_node_u2 = nullptr;        // [2n] (pred1, pred2)
  uint32_t* d_extra3_packed = nullptr; // [n_extra3] 3rd+ producer pairs, u | w << 16
  int32_t n_extra3 = 0;
  int32_t* d_out_off = nullptr;        // [n+1] fanout(v), edge order
  int32_t* d_out_edges = nullptr;      // [E]
  // joint-mode pair tables (built on first use, k_joint.cu)
  int2* d_joint_mul = nullptr;
  uint32_t* d_joint_ar = nullptr;
  uint32_t* d_joint_art = nullptr;
  int joint_ar_words = 0, joint_art_words = 0;
  int score_j = 0;                   // nodes per thread held in registers (0 = loop variant)
  int score_threads = 1024;
  int score_kc = 1;                  // candidates per CTA iteration (register variant)
  int score_warps = 0;               // >0: warp-per-candidate variant, warps per CTA
  int score_wp = 1;                  // its per-lane scan chunk (odd)
  int score_p = 1;                   // blocked scan chunk per thread (odd)

  // first node that misses a timestep in realized_lifetimes is searched on
  // the host in reference order; keep the CSR on the host too.
  std::vector<int32_t> h_edge_src;
  std::vector<int64_t> h_sink_off;
  std::vector<int32_t> h_sinks;
  std::vector<uint64_t> h_edge_size;

  bool smem_resident = false;
  size_t score_smem_bytes = 0;

  // node-partitioned large-graph scorer (mp_parts.cpp, k_score_parts.cuh)
  struct Parts {
    int32_t P = 0, nchunks = 0, nb_max = 0, nslots = 0, seg = 0;
    int32_t n_slot_init = 0, n_xfree = 0, n_cross_pairs = 0, n_cross_dyn = 0;
    size_t smem = 0;
    void* d_desc = nullptr;
    uint32_t* d_ctab = nullptr;
    uint8_t* d_xtab = nullptr;
    uint16_t* d_p1 = nullptr;
    uint32_t *d_intra = nullptr, *d_xput = nullptr, *d_xchk = nullptr, *d_xmax = nullptr;
    uint32_t *d_dyn4 = nullptr, *d_xfree = nullptr;
    int32_t* d_slot_init = nullptr;
  } parts;
  bool use_parts = false;
};

namespace mpb {

// Kernel launchers (k_*.cu). All stream-ordered, no synchronisation.
mp_status launch_score(const mp_graph* g, const int32_t* d_orders, int64_t num_orders,
                       uint64_t* d_peak, int32_t* d_peak_step, uint8_t* d_valid,
                       uint64_t* d_bytes /* [C][n] or null */,
                       uint64_t* d_key /* fused argmin key or null */, int64_t index_base,
                       cudaStream_t st,
                       int ofmt = 0 /* kOrdI32, or host-packed kOrdU16 / kOrdU24 */);
// the fused scorer reads 16-bit orders for this graph (register-slot variant, n < 65535)
bool score_takes_u16(const mp_graph* g);
// Order element formats of launch_score: the reference's int32, or the host-buffer
// call's wire formats (uint16 for the register-slot scorer, 3-byte ids for the
// node-partitioned one; both map out-of-range ids to an out-of-range value).
constexpr int kOrdI32 = 0, kOrdU16 = 1, kOrdU24 = 2;
bool score_takes_u24(const mp_graph* g);
size_t score_scratch_bytes(const mp_graph* g, int64_t num_orders);
mp_status score_configure(mp_graph* g);

mp_status launch_lifetimes(const mp_graph* g, const int32_t* d_order, int64_t order_len,
                           int32_t* d_lo, int32_t* d_hi, int32_t* d_valid, int32_t* d_pos_scratch,
                           cudaStream_t st);
mp_status launch_realized(const mp_graph* g, const int32_t* d_timestep_of, int32_t horizon,
                          int32_t* d_lo, int32_t* d_hi, int32_t* d_missing, cudaStream_t st);
mp_status launch_timeline(int32_t num_edges, const int32_t* d_lo, const int32_t* d_hi,
                          const uint64_t* d_size, int32_t horizon, uint64_t* d_bytes,
                          uint64_t* d_peak_rs, int32_t* d_peak_step, int64_t* d_diff_scratch,
                          cudaStream_t st);
// out3 = {best index + base or -1, best peak, packed key or UINT64_MAX}
mp_status launch_argmin(const uint64_t* d_peak, const uint8_t* d_valid, int64_t num_orders,
                        int64_t index_base, uint64_t* d_out3, cudaStream_t st);

// Pairwise sweeps. mode 0 = overlap pairs (a6), mode 1 = address conflicts (a11).
struct PairArgs {
  int32_t num_edges = 0;
  const int32_t* lo = nullptr;
  const int32_t* hi = nullptr;
  const uint64_t* size = nullptr;
  const uint8_t* mask = nullptr;   // pinned (mode 0) / has_addr (mode 1)
  const uint64_t* addr = nullptr;  // mode 1
  int mode = 0;
  int64_t row_begin = 0;
  int64_t row_end = 0;
};
size_t pairs_scratch_bytes(const PairArgs& a, int num_sms);
// Count pass + scan: d_row_off[rows+1]; the total stays in device memory
// (pairs_device_total) and is also copied to *h_total (sync) when h_total != NULL.
// Mode 0 counts from sorted column tiles (no O(E^2) sweep), mode 1 sweeps.
mp_status pairs_count(const PairArgs& a, int num_sms, void* d_scratch, int64_t* d_row_off,
                      int64_t* h_total, cudaStream_t st);
int64_t* pairs_device_total(const PairArgs& a, int num_sms, void* d_scratch);
// Fill pass using d_row_off from pairs_count; writes only the first `cap` pairs.
mp_status pairs_fill(const PairArgs& a, int num_sms, void* d_scratch, const int64_t* d_row_off,
                     int32_t* d_pairs, cudaStream_t st, int64_t cap = INT64_MAX);
// K5 placement (k_place.cu): preallocate_pyramid / greedy_pack / peak_mem per problem.
constexpr int kPlaceMaxEntries = 8192;  // placed tensors per problem (shared memory)
constexpr int kPlaceBigMaxEdges = (1 << 18) - 1;  // global-memory variant (two 512-ary levels)
struct PlaceArgs {
  int32_t num_edges = 0;
  int64_t num_problems = 0;
  const int32_t* lo = nullptr;         // [B][E]
  const int32_t* hi = nullptr;         // [B][E]
  const uint64_t* size = nullptr;      // [E]
  const int32_t* id_rank = nullptr;    // [E] or null (edge index order)
  const uint8_t* fixed = nullptr;      // [E] preplaced map or null
  const uint64_t* fixed_addr = nullptr;
  int pyramid = 0;                     // fixed = preallocate_pyramid(lifetimes)
  int pyramid_only = 0;                // stop after the pyramid
  uint64_t* addr = nullptr;            // [B][E]
  uint8_t* has_addr = nullptr;         // [B][E]
  uint64_t* peak_mem = nullptr;        // [B] or null
  uint64_t* pyramid_base = nullptr;    // [B] or null
  int cap = 0;                         // set by launch_place
  const int32_t* pyr_order = nullptr;  // [B][E] set by launch_place (global-memory variant)
};
size_t place_smem_bytes(int num_edges);
mp_status launch_place(const PlaceArgs& a, mp_ctx* ctx, cudaStream_t st);
// Batched plans (k_plans.cu): lifetimes per candidate order, the pairwise
// address check per plan, the first-minimum key over feasible plans.
size_t lifetimes_batch_smem(int32_t n);
// ... and for graphs past the shared-memory kernels (per-candidate K1, per-plan K4 sweep)
mp_status launch_lifetimes_large(const mp_graph* g, const int32_t* d_orders, int64_t C,
                                 int32_t* d_lo, int32_t* d_hi, int32_t* d_valid32,
                                 uint8_t* d_valid, int32_t* d_pos, cudaStream_t st);
mp_status launch_plan_check_large(mp_ctx* ctx, int64_t C, int32_t E, const int32_t* d_lo,
                                  const int32_t* d_hi, const uint64_t* d_size,
                                  const uint8_t* d_has, const uint64_t* d_addr,
                                  const uint8_t* d_valid, uint32_t* d_nviol, uint64_t* d_peak_mem,
                                  int64_t* d_row_off, cudaStream_t st);
size_t plan_check_smem(int32_t E);
mp_status launch_lifetimes_batch(const mp_graph* g, const int32_t* d_orders, int64_t C,
                                 int32_t* d_lo, int32_t* d_hi, uint8_t* d_valid, cudaStream_t st);
mp_status launch_plan_check(const mp_ctx* ctx, int64_t C, int32_t E, const int32_t* d_lo,
                            const int32_t* d_hi, const uint64_t* d_size, const uint8_t* d_has,
                            const uint64_t* d_addr, const uint8_t* d_valid, uint32_t* d_nviol,
                            uint64_t* d_peak_mem, cudaStream_t st);
mp_status launch_plan_key(int64_t C, const uint8_t* d_valid, const uint32_t* d_nviol,
                          const uint64_t* d_peak_mem, int64_t index_base, uint64_t* d_key,
                          cudaStream_t st);
// K8 joint-mode pair set (k_joint.cu): encode_joint's pair loop with edge_precedes.
struct JointArgs {
  int32_t E = 0;
  int filter = 1;
  const uint64_t* size = nullptr;
  const int32_t* src = nullptr;
  const int2* mul = nullptr;           // [E] compute_bounds' multiplicity windows
  const uint32_t* ar = nullptr;        // [E][ar_words]  AR(e): nodes every sink of e reaches
  const uint32_t* art = nullptr;       // [n][art_words] transposed
  int ar_words = 0, art_words = 0;
};
mp_status launch_joint(const JointArgs& a, int num_sms, int64_t* d_row_cnt,
                       const int64_t* d_row_off, int2* d_pairs, cudaStream_t st);
// Descendant bitsets are built on the host (n^2 / 8 bytes), AR uploaded and
// transposed on the device; both bounded by kJointMaxTableBytes.
constexpr int32_t kJointMaxNodes = 1 << 18;
constexpr size_t kJointMaxTableBytes = size_t{6} << 30;
// ARt[v][e / 32] bit e % 32 = AR[e][v / 32] bit v % 32, 32 x 32 blocks by ballots
mp_status launch_joint_transpose(const uint32_t* d_ar, int32_t E, int32_t n, int ar_words,
                                 int art_words, uint32_t* d_art, cudaStream_t st);

// K7 LP row emission (k_lp.cu): write_lp text of encode_addresses' pair rows.
struct LpArgs {
  int32_t E = 0;
  int64_t P = 0;                        // overlapping pairs
  const int2* pairs = nullptr;          // [P] (i, j), i < j
  const uint64_t* size = nullptr;       // [E]
  const uint8_t* pinned = nullptr;      // [E] or null
  const uint64_t* pinned_addr = nullptr;
  const char* names = nullptr;          // sanitized edge ids, concatenated
  const int64_t* name_off = nullptr;    // [E+1]
  long long M = 0;                      // big-M = Graph::total_bytes (encode.cpp:325)
  int64_t* row_len = nullptr;           // [P]
  int64_t* bin_len = nullptr;           // [P]
  const int64_t* row_off = nullptr;     // [P] exclusive scan of row_len
  const int64_t* bin_off = nullptr;
};
mp_status launch_lp_len(const LpArgs& a, int num_sms, cudaStream_t st);
mp_status launch_lp_write(const LpArgs& a, char* d_rows, char* d_bins, int num_sms,
                          cudaStream_t st);
size_t lp_scan_scratch(int64_t n);
mp_status scan_exclusive_i64(const int64_t* d_in, int64_t n, int64_t* d_out, int64_t* d_sums,
                             int64_t* d_total, cudaStream_t st);

// K6 arena baseline (k_arena.cu): run_baseline per candidate order.
struct ArenaArgs {
  int32_t n = 0, E = 0, cap = 0;       // cap: block-list capacity (set by launch_arena)
  int retry = 0;                       // second pass: only candidates marked overflowed
  int64_t num_orders = 0;
  const int32_t* orders = nullptr;     // [B][n]
  const int32_t* edge_src = nullptr;
  const int64_t* sink_off = nullptr;
  const int32_t* sinks = nullptr;
  const uint64_t* edge_size = nullptr;
  const uint32_t* edge_size32 = nullptr;  // size / scale (null: 64-bit block sizes)
  uint64_t scale = 1;
  const int32_t* out_off = nullptr;    // fanout lists
  const int32_t* out_edges = nullptr;
  int best_fit = 0;
  uint64_t* mr_peak = nullptr;         // [B]
  uint64_t* rs_at_peak = nullptr;      // [B]
  double* frag = nullptr;              // [B]
  uint8_t* valid = nullptr;            // [B]
};
constexpr int kArenaCap = 1024;       // first-pass block-list capacity
size_t arena_smem_bytes(int n, int E, int cap, int size_bytes = 8, int edge_index = 1);
mp_status launch_arena(const ArenaArgs& a, const mp_ctx* ctx, cudaStream_t st);
mp_status launch_peak_mem(int32_t num_edges, const uint64_t* d_size, const uint8_t* d_has,
                          const uint64_t* d_addr, uint64_t* d_out, cudaStream_t st);

}  // namespace mpb
