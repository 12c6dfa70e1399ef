/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.
 *
 * Plain-C restatement of the reference planner's data-parallel hot path
 * (memplan, /root/reference/proj). Each function cites the reference
 * file:line it follows. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library (oracle/_build/liboracle.so).
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by the reference itself
 * (oracle/_ref/libmemplan_ref.so, tests/golden/make_golden.py) and against
 * the reference's own known-answer tests.
 *
 * Graph representation (the reference's Graph, graph.hpp:62-127, flattened):
 *   n nodes, E edges; edge_src[E]; sink_off[E+1] (int64); sinks[S];
 *   edge_size[E] (0 for control edges, graph.cpp:89-93).
 */
#ifndef MEMPLAN_ORACLE_H_
#define MEMPLAN_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t n;
  int32_t num_edges;
  const int32_t* edge_src;
  const int64_t* sink_off;
  const int32_t* sinks;
  const uint64_t* edge_size;
} or_graph;

/* graph.cpp:239-254 */
int or_is_topological_order(const or_graph* g, const int32_t* order, int64_t len);
/* schedule.cpp:23-31 -> 0 ok, 1 InvalidOrder; pos is 1-based. */
int or_positions_of(const or_graph* g, const int32_t* order, int64_t len, int32_t* pos);
/* schedule.cpp:33-50 */
int or_lifetimes_from_order(const or_graph* g, const int32_t* order, int64_t len,
                            int32_t* lo, int32_t* hi);
/* schedule.cpp:69-79 (literal O(sum of lifetime lengths) loop) */
int or_resident_bytes_per_step(const or_graph* g, const int32_t* order, int64_t len,
                               uint64_t* out);
/* schedule.cpp:81-88 */
int or_peak_resident_bytes(const or_graph* g, const int32_t* order, int64_t len,
                           uint64_t* peak);
/* plan.cpp:122-143: bytes[horizon] (may be NULL), peak_rs, peak_step */
void or_timeline_from_lifetimes(const or_graph* g, const int32_t* lo, const int32_t* hi,
                                int32_t horizon, uint64_t* bytes, uint64_t* peak_rs,
                                int32_t* peak_step);
/* plan.cpp:101-120; timestep_of[v]==0 means absent. Returns 0 ok, or
 * 1 + (node index that is missing) encoded as -(v+1) in *missing. */
int or_realized_lifetimes(const or_graph* g, const int32_t* timestep_of, int32_t horizon,
                          int32_t* lo, int32_t* hi, int32_t* missing);
/* encode.cpp:329-357 with the filter reduced to interval intersection
 * (exact for lifetimes realized from a topological order).
 * Pairs in lexicographic (i,j) order; pairs==NULL counts only. */
int64_t or_overlap_pairs(int32_t num_edges, const int32_t* lo, const int32_t* hi,
                         const uint64_t* size, const uint8_t* pinned,
                         int32_t* pairs, int64_t cap);
/* Per-row pair counts (row i = number of j>i forming a pair with i) and a
 * 64-bit FNV-1a hash over each row's j list, for parity at scale. */
void or_overlap_row_stats(int32_t num_edges, const int32_t* lo, const int32_t* hi,
                          const uint64_t* size, const uint8_t* pinned,
                          int64_t row_begin, int64_t row_end,
                          int64_t* row_count, uint64_t* row_hash);
/* plan.cpp:390-404: conflicting pairs among data edges with an address. */
int64_t or_validate_pairs(int32_t num_edges, const int32_t* lo, const int32_t* hi,
                          const uint64_t* size, const uint8_t* has_addr,
                          const uint64_t* addr, int32_t* viol, int64_t cap);
/* pipeline.cpp:146-160 */
int or_addresses_feasible(int32_t num_edges, const int32_t* lo, const int32_t* hi,
                          const uint64_t* size, const uint8_t* has_addr,
                          const uint64_t* addr);
/* placement.cpp:64-67 */
double or_fragmentation(uint64_t mr, uint64_t rs);
/* pipeline.cpp:270-275 */
uint64_t or_peak_mem(int32_t num_edges, const uint64_t* size, const uint8_t* has_addr,
                     const uint64_t* addr);

/* preallocate_pyramid (placement.cpp:25-62): taken[e] = 1 and addr[e] = its base
 * for the picked edges; returns reserved_base. id_rank[e] orders edge ids
 * (byte-lexicographic) for the last tie-break (placement.cpp:48-50). */
uint64_t or_preallocate_pyramid(int32_t num_edges, const int32_t* lo, const int32_t* hi,
                                const uint64_t* size, const int32_t* id_rank, uint8_t* taken,
                                uint64_t* addr);
/* greedy_pack (placement.cpp:182-204) with the preplaced map given as
 * fixed[e] / addr[e] (in/out): on return has[e] = 1 for every placed edge. */
void or_greedy_pack(int32_t num_edges, const int32_t* lo, const int32_t* hi, const uint64_t* size,
                    const uint8_t* fixed, uint64_t* addr, uint8_t* has);

/* run_baseline (placement.cpp:150-180) with the free-list Arena of
 * placement.cpp:69-148, literally. best_fit: FitPolicy::kBestFit. Returns 0, or
 * 1 for InvalidOrder (lifetimes_from_order throws). */
int or_run_baseline(const or_graph* g, const int32_t* order, int64_t len, int best_fit,
                    uint64_t* mr_peak, uint64_t* rs_at_peak, double* frag);

/* The pair loop of encode_joint (encode.cpp:401-408): data edges a < b (edge
 * order), skipped when filter != 0 and edge_precedes holds either way
 * (analysis.cpp:94-113) with compute_bounds (analysis.cpp:11-62) and a memoised
 * ancestor search as ReachabilityCache (analysis.cpp:79-92). Two-phase: pairs may
 * be NULL; returns the count (-1 on a cycle). */
int64_t or_joint_pairs(const or_graph* g, int filter, int32_t* pairs, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* MEMPLAN_ORACLE_H_ */
