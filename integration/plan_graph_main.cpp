// The reference's planning entry point, plan_graph (proj/src/pipeline.cpp:296-324),
// driven from the command line - built twice by integration/Makefile: against the
// unmodified reference objects (plan_graph_ref) and against pipeline.cpp with
// integration/pipeline_b200.patch applied (plan_graph_b200: its hot-path call
// sites go through include/memplan_b200.hpp on a B200). Both print the same
// record, so tests/test_gpu_integration.py compares them byte for byte.
//
//   plan_graph_{ref,b200} plan  <graph.json>...   PlanResult per graph
//   plan_graph_{ref,b200} peak  <graph.json> <reps>
//       latency of the call site pipeline.cpp:297-302 (peak_resident_bytes of the
//       program order): first call (B200: includes the upload and host analysis)
//       and the mean of `reps` further calls, in microseconds
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>

#include "memplan/errors.hpp"
#include "memplan/graph_io.hpp"
#include "memplan/pipeline.hpp"
#include "memplan/plan.hpp"
#include "memplan/schedule.hpp"
#ifdef MEMPLAN_WITH_B200
#include "memplan_b200.hpp"
#endif

namespace {
// program order exactly as pipeline.cpp:38-45 builds it (internal there): node
// order when it is topological, else the canonical topological order
std::vector<memplan::NodeIndex> program_order(const memplan::Graph& g) {
  std::vector<memplan::NodeIndex> order(g.num_nodes());
  for (int v = 0; v < g.num_nodes(); ++v) order[v] = v;
  if (g.num_nodes() == 0 || memplan::is_topological_order(g, order)) return order;
  return memplan::topological_order(g);
}

std::uint64_t peak_call(const memplan::Graph& g) {
#ifdef MEMPLAN_WITH_B200
  static memplan_b200::Planner planner(0);
  return planner.peak_resident_bytes(g, program_order(g));
#else
  return memplan::peak_resident_bytes(g, program_order(g));
#endif
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s plan <graph.json>... | peak <graph.json> <reps>\n", argv[0]);
    return 2;
  }
  const std::string mode = argv[1];
  try {
    if (mode == "plan") {
      for (int i = 2; i < argc; ++i) {
        const memplan::Graph g = memplan::load_graph_file(argv[i]);
        const memplan::PlanResult r = memplan::plan_graph(g);
        std::cout << "== " << argv[i] << "\n"
                  << "program_order_peak " << r.program_order_peak << "\n"
                  << "savings_percent " << r.savings_percent << "\n"
                  << "control_edges_added " << r.control_edges_added << "\n"
                  << "timed_out " << r.timed_out << "\n"
                  << memplan::save_plan(r.plan) << "\n"
                  << "validate " << memplan::validate_plan(r.plan, g).ok() << "\n";
      }
      return 0;
    }
    if (mode == "peak" && argc == 4) {
      const memplan::Graph g = memplan::load_graph_file(argv[2]);
      const int reps = std::atoi(argv[3]);
      auto t0 = std::chrono::steady_clock::now();
      std::uint64_t p = peak_call(g);
      auto t1 = std::chrono::steady_clock::now();
      for (int k = 0; k < reps; ++k) p ^= peak_call(g) ^ p;
      auto t2 = std::chrono::steady_clock::now();
      std::printf("{\"peak\": %llu, \"first_us\": %.1f, \"cached_us\": %.1f}\n",
                  (unsigned long long)peak_call(g),
                  std::chrono::duration<double, std::micro>(t1 - t0).count(),
                  std::chrono::duration<double, std::micro>(t2 - t1).count() / (reps > 0 ? reps : 1));
      return 0;
    }
  } catch (const memplan::Error& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 3;
  }
  return 2;
}
