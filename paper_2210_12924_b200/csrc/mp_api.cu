// C ABI of memplan_b200 (include/memplan_b200.h): contexts, graph upload
// with the derived scoring tables, and the host-buffer / device-buffer entry
// points that launch the kernels in k_score.cu, k_lifetimes.cu, k_pairs.cu.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <thread>
#include <unordered_set>
#include <cctype>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "mp_internal.h"
#include "mp_parts.h"
#include "mp_prep.h"

namespace mpb {

namespace {
thread_local std::string g_err;
const char* kInvalidOrderMsg = "InvalidOrder: sequence is not a topological order of the graph";
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }

mp_status cuda_status(cudaError_t e, const char* what) {
  set_error(std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")");
  cudaGetLastError();  // clear sticky-free errors
  return e == cudaErrorMemoryAllocation ? MP_E_OOM : MP_E_CUDA;
}

mp_status Scratch::reserve(size_t want) {
  if (want <= bytes && ptr) return MP_OK;
  if (ptr) {
    cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  size_t b = want + want / 4 + 4096;
  MP_CUDA(cudaMalloc(&ptr, b));
  bytes = b;
  return MP_OK;
}

Scratch::~Scratch() {
  if (ptr) cudaFree(ptr);
}

// Bump allocator over one scratch slot (256-byte aligned pieces).
struct Carver {
  char* base;
  size_t at = 0;
  explicit Carver(void* p) : base(static_cast<char*>(p)) {}
  template <typename T>
  T* take(size_t count) {
    T* p = reinterpret_cast<T*>(base + at);
    at += (count * sizeof(T) + 255) & ~size_t(255);
    return p;
  }
  static size_t size_of(std::initializer_list<size_t> bytes) {
    size_t s = 0;
    for (size_t b : bytes) s += (b + 255) & ~size_t(255);
    return s + 256;
  }
};

struct DeviceGuard {
  explicit DeviceGuard(int dev) { cudaSetDevice(dev); }
};

mp_status invalid_order() {
  set_error(kInvalidOrderMsg);
  return MP_E_INVALID_ORDER;
}

mp_status invalid_arg(const std::string& what) {
  set_error("InvalidArgument: " + what);
  return MP_E_INVALID_ARG;
}

template <typename T>
mp_status upload(T** dst, const T* src, size_t count, cudaStream_t st) {
  *dst = nullptr;
  if (count == 0) return MP_OK;
  MP_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), count * sizeof(T)));
  MP_CUDA(cudaMemcpyAsync(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice, st));
  return MP_OK;
}

}  // namespace mpb

using namespace mpb;

namespace {
// A graph is bound to the context (device) it was uploaded to: a graph
// from another context would launch kernels on one device over another's tables.
mp_status same_ctx(const mp_ctx* ctx, const mp_graph* g) {
  if (ctx && g && g->ctx != ctx) return invalid_arg("graph belongs to another context");
  return MP_OK;
}
}  // namespace

extern "C" {

int mp_abi_version(void) { return MP_ABI_VERSION; }

const char* mp_status_string(mp_status s) {
  switch (s) {
    case MP_OK: return "MP_OK";
    case MP_E_INVALID_ORDER: return "MP_E_INVALID_ORDER";
    case MP_E_BAD_GRAPH: return "MP_E_BAD_GRAPH";
    case MP_E_INVALID_ARG: return "MP_E_INVALID_ARG";
    case MP_E_CUDA: return "MP_E_CUDA";
    case MP_E_OOM: return "MP_E_OOM";
    case MP_E_CAPACITY: return "MP_E_CAPACITY";
    case MP_E_NO_DEVICE: return "MP_E_NO_DEVICE";
  }
  return "MP_E_UNKNOWN";
}

const char* mp_last_error(void) { return g_err.c_str(); }

mp_status mp_ctx_create(int device, mp_ctx** out) {
  if (!out) return invalid_arg("out is null");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    set_error("memplan_b200: no CUDA device visible; there is no CPU fallback");
    return MP_E_NO_DEVICE;
  }
  if (device < 0 || device >= count) return invalid_arg("device index out of range");
  cudaDeviceProp prop;
  MP_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_error("memplan_b200: device " + std::to_string(device) + " is sm_" +
              std::to_string(prop.major) + std::to_string(prop.minor) +
              "; this library is built for sm_100a only");
    return MP_E_NO_DEVICE;
  }
  DeviceGuard guard(device);
  auto* ctx = new mp_ctx();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  ctx->max_smem_optin = (size_t)optin;
  cudaError_t ce = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (ce == cudaSuccess) ce = cudaMalloc(reinterpret_cast<void**>(&ctx->d_small), 256);
  if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
  for (int i = 0; i < mp_ctx::kPipeChunks && ce == cudaSuccess; ++i)
    ce = cudaEventCreateWithFlags(&ctx->ev_h2d[i], cudaEventDisableTiming);
  if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&ctx->ev_start, cudaEventDisableTiming);
  if (ce == cudaSuccess) ce = cudaMallocHost(reinterpret_cast<void**>(&ctx->h_small), 64);
  for (int i = 0; i < 2 && ce == cudaSuccess; ++i)
    ce = cudaEventCreateWithFlags(&ctx->ev_d2h[i], cudaEventDisableTiming);
  if (ce != cudaSuccess) {
    mp_status s = cuda_status(ce, "mp_ctx_create");
    delete ctx;
    return s;
  }
  ctx->stream = ctx->own_stream;
  *out = ctx;
  return MP_OK;
}

mp_status mp_ctx_destroy(mp_ctx* ctx) {
  if (!ctx) return MP_OK;
  DeviceGuard guard(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->d_small) cudaFree(ctx->d_small);
  for (cudaEvent_t e : ctx->ev_h2d)
    if (e) cudaEventDestroy(e);
  if (ctx->ev_start) cudaEventDestroy(ctx->ev_start);
  if (ctx->h_small) cudaFreeHost(ctx->h_small);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  if (ctx->h_bounce) cudaFreeHost(ctx->h_bounce);
  for (cudaEvent_t e : ctx->ev_d2h)
    if (e) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return MP_OK;
}

mp_status mp_ctx_set_stream(mp_ctx* ctx, void* stream) {
  if (!ctx) return invalid_arg("ctx is null");
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  return MP_OK;
}

mp_status mp_ctx_synchronize(mp_ctx* ctx) {
  if (!ctx) return invalid_arg("ctx is null");
  DeviceGuard guard(ctx->device);
  MP_CUDA(cudaStreamSynchronize(ctx->stream));
  return MP_OK;
}

// ---- graph upload -----------------------------------------------------------
mp_status mp_graph_upload(mp_ctx* ctx, const mp_csr* csr, mp_graph** out) {
  if (!ctx || !csr || !out) return invalid_arg("null argument");
  *out = nullptr;
  const int32_t n = csr->num_nodes, E = csr->num_edges;
  if (n < 0 || E < 0) return invalid_arg("negative graph dimensions");
  if (E > 0 && (!csr->edge_src || !csr->sink_off || !csr->edge_size))
    return invalid_arg("edge arrays are null");
  if (E > 0 && csr->sink_off[0] != 0) {
    set_error("InvalidStructure: sink_off[0] must be 0");
    return MP_E_BAD_GRAPH;
  }
  const int64_t S = E > 0 ? csr->sink_off[E] : 0;
  if (S > 0 && !csr->sinks) return invalid_arg("sinks is null");

  auto* g = new mp_graph();
  g->ctx = ctx;
  g->n = n;
  g->E = E;
  g->S = S;
  g->h_edge_src.assign(csr->edge_src, csr->edge_src + E);
  g->h_sink_off.assign(csr->sink_off, csr->sink_off + (E > 0 ? E + 1 : 0));
  if (E == 0) g->h_sink_off.assign(1, 0);
  g->h_sinks.assign(csr->sinks, csr->sinks + S);
  g->h_edge_size.assign(csr->edge_size, csr->edge_size + E);

  // Structural checks the kernels rely on (Graph::build, graph.cpp:82-128).
  uint64_t total = 0;
  const uint64_t cap = uint64_t{1} << 62;
  std::vector<int32_t> seen_stamp(n, -1);
  for (int32_t e = 0; e < E; ++e) {
    const int32_t s = g->h_edge_src[e];
    const int64_t a = g->h_sink_off[e], b = g->h_sink_off[e + 1];
    std::string err;
    if (s < 0 || s >= n) err = "DanglingEndpoint: edge #" + std::to_string(e) + " has unknown source";
    else if (b < a || b > S) err = "InvalidStructure: sink offsets are not monotone";
    for (int64_t k = a; err.empty() && k < b; ++k) {
      const int32_t w = g->h_sinks[k];
      if (w < 0 || w >= n) err = "DanglingEndpoint: edge #" + std::to_string(e) + " has unknown sink";
      else if (seen_stamp[w] == e) err = "InvalidStructure: edge #" + std::to_string(e) + " lists a sink twice";
      else seen_stamp[w] = e;
    }
    const uint64_t sz = g->h_edge_size[e];
    if (err.empty() && (sz >= cap || total + sz >= cap))
      err = "InvalidStructure: total tensor bytes exceed the supported range";
    if (!err.empty()) {
      set_error(err);
      delete g;
      return MP_E_BAD_GRAPH;
    }
    total += sz;
  }
  g->total_bytes = total;

  // Scoring tables (transitive reduction, static last consumers, gcd scale).
  ScorePrep P;
  prepare_scoring(n, E, g->h_edge_src.data(), g->h_sink_off.data(), g->h_sinks.data(),
                  g->h_edge_size.data(), &P);
  g->n_preds = P.num_reduced_preds;
  g->n_extra = (int32_t)P.extra3_u.size();
  g->n_dyn = (int32_t)P.dyn_size.size();
  g->n_dyn_sinks = (int32_t)P.dyn_sinks.size();
  for (size_t d = 0; d + 1 < P.dyn_off.size(); ++d)
    g->dyn_max_sinks = std::max(g->dyn_max_sinks, P.dyn_off[d + 1] - P.dyn_off[d]);
  g->scale = P.scale;
  g->narrow = P.narrow;
  g->mid32 = P.mid32 && !std::getenv("MP_SCORE_NO_MID");
  g->tiny8 = P.tiny8;
  g->tiny4 = P.tiny4;
  g->exact_reach = P.exact_reach;

  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  mp_status s = MP_OK;
  auto up = [&](mp_status r) {
    if (s == MP_OK) s = r;
  };
  up(upload(&g->d_edge_src, g->h_edge_src.data(), (size_t)E, st));
  up(upload(&g->d_sink_off, g->h_sink_off.data(), (size_t)E + 1, st));
  up(upload(&g->d_sinks, g->h_sinks.data(), (size_t)S, st));
  up(upload(&g->d_edge_size, g->h_edge_size.data(), (size_t)E, st));
  up(upload(&g->d_node_x, P.node_x.data(), P.node_x.size(), st));
  up(upload(&g->d_node_f, P.node_f.data(), P.node_f.size(), st));
  up(upload(&g->d_pred1, P.pred1.data(), P.pred1.size(), st));
  // the node-table scorer checks pred1 and pred2 in node space: its flat list is the 3rd+
  up(upload(&g->d_extra_u, P.extra3_u.data(), P.extra3_u.size(), st));
  up(upload(&g->d_extra_w, P.extra3_w.data(), P.extra3_w.size(), st));
  up(upload(&g->d_dyn_off, P.dyn_off.data(), P.dyn_off.size(), st));
  up(upload(&g->d_dyn_sinks, P.dyn_sinks.data(), P.dyn_sinks.size(), st));
  up(upload(&g->d_dyn_size, P.dyn_size.data(), P.dyn_size.size(), st));
  up(upload(&g->d_node_rec32, P.node_rec32.data(), P.node_rec32.size(), st));
  up(upload(&g->d_node_u2, P.node_u2.data(), P.node_u2.size(), st));
  up(upload(&g->d_extra3_packed, P.extra3_packed.data(), P.extra3_packed.size(), st));
  g->n_extra3 = (int32_t)P.extra3_packed.size();
  if (g->dyn_max_sinks <= 4 && g->n_dyn > 0) {
    std::vector<int32_t> s4(4 * (size_t)g->n_dyn, -1);
    for (int32_t d = 0; d < g->n_dyn; ++d)
      for (int32_t k = P.dyn_off[d]; k < P.dyn_off[d + 1]; ++k)
        s4[4 * (size_t)d + (k - P.dyn_off[d])] = P.dyn_sinks[k];
    up(upload(&g->d_dyn_sink4, s4.data(), s4.size(), st));
  }
  std::vector<uint32_t> size32;
  if (g->narrow) {
    size32.resize((size_t)E);
    for (int32_t e = 0; e < E; ++e) size32[e] = (uint32_t)(g->h_edge_size[e] / g->scale);
    up(upload(&g->d_edge_size32, size32.data(), size32.size(), st));
  }
  up(upload(&g->d_out_off, P.out_off.data(), P.out_off.size(), st));
  up(upload(&g->d_out_edges, P.out_edges.data(), P.out_edges.size(), st));
  // Large tiny4 graphs: plan the node partition of the shared-memory scorer
  // (MP_SCORE_PARTS forces it on any tiny4 graph, MP_PARTS_CHUNKS caps the chunks
  // per part - both for tests; MP_SCORE_NO_PARTS keeps the scratch scorer).
  const bool scratch_knob = std::getenv("MP_SCORE_NO_PARTS") || std::getenv("MP_SCORE_POS64") ||
                            std::getenv("MP_SCORE_WIDE_XF") || std::getenv("MP_SCORE_NO_TINY4");
  if (s == MP_OK && P.tiny4 && n > 0 && !scratch_knob &&
      (n >= kPartsMinNodes || std::getenv("MP_SCORE_PARTS"))) {
    const char* mc = std::getenv("MP_PARTS_CHUNKS");
    PartPlan pp;
    if (plan_parts(P, ctx->max_smem_optin, mc ? std::atoi(mc) : 0, &pp)) {
      auto& Q = g->parts;
      Q.P = pp.P;
      Q.nchunks = pp.nchunks;
      Q.nb_max = pp.nb_max;
      Q.nslots = pp.nslots;
      Q.n_slot_init = (int32_t)pp.slot_init_max.size();
      Q.n_xfree = (int32_t)(pp.xfree.size() / 2);
      Q.n_cross_pairs = pp.n_cross_pairs;
      Q.n_cross_dyn = pp.n_cross_dyn;
      Q.seg = ((n + 32 * 512 - 1) / (32 * 512)) * 512;  // per-warp segment: 32 lane chunks of 16-byte multiples
      Q.smem = parts_smem_bytes(pp);
      std::vector<int32_t> desc(pp.desc.size() * (sizeof(PartDesc) / 4));
      std::memcpy(desc.data(), pp.desc.data(), desc.size() * 4);
      int32_t* dd = nullptr;
      up(upload(&dd, desc.data(), desc.size(), st));
      Q.d_desc = dd;
      up(upload(&Q.d_ctab, pp.ctab.data(), pp.ctab.size(), st));
      up(upload(&Q.d_xtab, pp.xtab.data(), pp.xtab.size(), st));
      up(upload(&Q.d_p1, pp.p1.data(), pp.p1.size(), st));
      up(upload(&Q.d_intra, pp.intra.data(), pp.intra.size(), st));
      up(upload(&Q.d_xput, pp.xput.data(), pp.xput.size(), st));
      up(upload(&Q.d_xchk, pp.xchk.data(), pp.xchk.size(), st));
      up(upload(&Q.d_xmax, pp.xmax.data(), pp.xmax.size(), st));
      up(upload(&Q.d_dyn4, pp.dyn4.data(), pp.dyn4.size(), st));
      up(upload(&Q.d_xfree, pp.xfree.data(), pp.xfree.size(), st));
      up(upload(&Q.d_slot_init, pp.slot_init_max.data(), pp.slot_init_max.size(), st));
      if (s == MP_OK) up(cudaStreamSynchronize(st) == cudaSuccess ? MP_OK : MP_E_CUDA);
    }
  }
  if (s == MP_OK) up(score_configure(g));
  if (s == MP_OK) {
    cudaError_t ce = cudaStreamSynchronize(st);  // host tables may go out of scope
    if (ce != cudaSuccess) s = cuda_status(ce, "mp_graph_upload");
  }
  if (s != MP_OK) {
    mp_graph_free(g);
    return s;
  }
  *out = g;
  return MP_OK;
}

mp_status mp_parts_plan_host(const mp_csr* csr, int32_t max_chunks, int64_t smem_budget,
                             int64_t* info) {
  if (!csr || !info || csr->num_nodes < 0 || csr->num_edges < 0) return invalid_arg("bad argument");
  ScorePrep P;
  prepare_scoring(csr->num_nodes, csr->num_edges, csr->edge_src, csr->sink_off, csr->sinks,
                  csr->edge_size, &P);
  PartPlan pp;
  const bool ok = plan_parts(P, (size_t)smem_budget, max_chunks, &pp);
  info[0] = ok ? pp.P : 0;
  info[1] = pp.nb_max;
  info[2] = pp.nslots;
  info[3] = pp.n_cross_pairs;
  info[4] = pp.n_cross_dyn;
  info[5] = ok ? (int64_t)parts_smem_bytes(pp) : 0;
  info[6] = P.tiny4 ? 1 : 0;
  return MP_OK;
}

mp_status mp_prep_host(const mp_csr* csr, int64_t* info, int32_t* pairs, int64_t cap) {
  if (!csr || !info || csr->num_nodes < 0 || csr->num_edges < 0 || cap < 0)
    return invalid_arg("bad argument");
  ScorePrep P;
  prepare_scoring(csr->num_nodes, csr->num_edges, csr->edge_src, csr->sink_off, csr->sinks,
                  csr->edge_size, &P);
  info[0] = P.num_reduced_preds;
  info[1] = (int64_t)P.dyn_size.size();
  info[2] = P.exact_reach ? 1 : 0;
  info[3] = P.tiny4 ? 1 : 0;
  info[4] = P.tiny8 ? 1 : 0;
  info[5] = P.narrow ? 1 : 0;
  info[6] = P.mid32 ? 1 : 0;
  if (pairs) {
    int64_t k = 0;
    for (int32_t w = 0; w < P.n && k < cap; ++w)
      if (P.pred1[w] >= 0) {
        pairs[2 * k] = P.pred1[w];
        pairs[2 * k + 1] = w;
        ++k;
      }
    for (size_t i = 0; i < P.extra_u.size() && k < cap; ++i, ++k) {
      pairs[2 * k] = P.extra_u[i];
      pairs[2 * k + 1] = P.extra_w[i];
    }
  }
  return MP_OK;
}

mp_status mp_graph_free(mp_graph* g) {
  if (!g) return MP_OK;
  DeviceGuard guard(g->ctx->device);
  void* ptrs[] = {g->d_edge_src, g->d_sink_off,  g->d_sinks,     g->d_edge_size,
                  g->d_node_x,   g->d_node_f,    g->d_pred1,     g->d_extra_u,
                  g->d_extra_w,  g->d_dyn_off,   g->d_dyn_sinks, g->d_dyn_size,
                  g->d_node_rec32, g->d_node_u2, g->d_extra3_packed,
                  g->d_out_off,  g->d_out_edges, g->d_dyn_sink4, g->d_joint_mul,
                  g->d_joint_ar, g->d_joint_art, g->d_edge_size32,
                  g->parts.d_desc, g->parts.d_ctab, g->parts.d_xtab, g->parts.d_p1, g->parts.d_intra,
                  g->parts.d_xput, g->parts.d_xchk, g->parts.d_xmax, g->parts.d_dyn4,
                  g->parts.d_xfree, g->parts.d_slot_init};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete g;
  return MP_OK;
}

mp_status mp_graph_get_info(const mp_graph* g, mp_graph_info* info) {
  if (!g || !info) return invalid_arg("null argument");
  info->num_nodes = g->n;
  info->num_edges = g->E;
  info->num_sinks = g->S;
  info->num_pred_pairs = g->n_preds;
  info->num_multi_sink = g->n_dyn;
  info->smem_resident = g->smem_resident ? 1 : 0;
  info->total_bytes = g->total_bytes;
  info->orders16 = score_takes_u16(g) && !std::getenv("MP_NO_PACK16")   ? 1
                   : score_takes_u24(g) && std::getenv("MP_PACK24")     ? 2
                                                                        : 0;
  info->score_variant = g->use_parts        ? MP_SCORER_PARTS
                        : g->score_warps > 0 ? MP_SCORER_WARP
                        : g->score_j > 0    ? MP_SCORER_REG
                        : g->smem_resident  ? MP_SCORER_SMEM
                                            : MP_SCORER_SCRATCH;
  return MP_OK;
}

// ---- lifetimes ------------------------------------------------------------------
mp_status mp_lifetimes_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_order, int64_t len,
                         int32_t* d_lo, int32_t* d_hi, int32_t* d_valid, void* stream) {
  MP_TRY(same_ctx(ctx, g));
  if (!ctx || !g || (len > 0 && !d_order) || !d_valid) return invalid_arg("null argument");
  DeviceGuard guard(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL: default stream
  MP_TRY(ctx->scratch[2].reserve(sizeof(int32_t) * ((size_t)g->n + 1)));
  return launch_lifetimes(g, d_order, len, d_lo, d_hi, d_valid,
                          static_cast<int32_t*>(ctx->scratch[2].ptr), st);
}

mp_status mp_lifetimes(mp_ctx* ctx, const mp_graph* g, const int32_t* order, int64_t len,
                       int32_t* lo, int32_t* hi) {
  MP_TRY(same_ctx(ctx, g));
  if (!ctx || !g || (len > 0 && !order) || (g->E > 0 && (!lo || !hi)))
    return invalid_arg("null argument");
  if (len != g->n) return invalid_order();
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t n = (size_t)g->n, E = (size_t)g->E;
  MP_TRY(ctx->scratch[0].reserve(Carver::size_of({4 * n, 4 * E, 4 * E, 4})));
  Carver cv(ctx->scratch[0].ptr);
  int32_t* d_order = cv.take<int32_t>(n);
  int32_t* d_lo = cv.take<int32_t>(E);
  int32_t* d_hi = cv.take<int32_t>(E);
  int32_t* d_valid = cv.take<int32_t>(1);
  if (n) MP_CUDA(cudaMemcpyAsync(d_order, order, 4 * n, cudaMemcpyHostToDevice, st));
  MP_TRY(mp_lifetimes_d(ctx, g, d_order, len, d_lo, d_hi, d_valid, st));
  int32_t valid = 0;
  MP_CUDA(cudaMemcpyAsync(&valid, d_valid, 4, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  if (!valid) return invalid_order();
  if (E) {
    MP_CUDA(cudaMemcpyAsync(lo, d_lo, 4 * E, cudaMemcpyDeviceToHost, st));
    MP_CUDA(cudaMemcpyAsync(hi, d_hi, 4 * E, cudaMemcpyDeviceToHost, st));
    MP_CUDA(cudaStreamSynchronize(st));
  }
  return MP_OK;
}

mp_status mp_realized_lifetimes(mp_ctx* ctx, const mp_graph* g, const int32_t* timestep_of,
                                int32_t horizon, int32_t* lo, int32_t* hi,
                                int32_t* missing_node) {
  MP_TRY(same_ctx(ctx, g));
  if (!ctx || !g || (g->n > 0 && !timestep_of) || (g->E > 0 && (!lo || !hi)))
    return invalid_arg("null argument");
  if (missing_node) *missing_node = -1;
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t n = (size_t)g->n, E = (size_t)g->E;
  MP_TRY(ctx->scratch[0].reserve(Carver::size_of({4 * n, 4 * E, 4 * E, 4})));
  Carver cv(ctx->scratch[0].ptr);
  int32_t* d_ts = cv.take<int32_t>(n);
  int32_t* d_lo = cv.take<int32_t>(E);
  int32_t* d_hi = cv.take<int32_t>(E);
  int32_t* d_bad = cv.take<int32_t>(1);
  if (n) MP_CUDA(cudaMemcpyAsync(d_ts, timestep_of, 4 * n, cudaMemcpyHostToDevice, st));
  const int32_t big = INT_MAX;
  MP_CUDA(cudaMemcpyAsync(d_bad, &big, 4, cudaMemcpyHostToDevice, st));
  MP_TRY(launch_realized(g, d_ts, horizon, d_lo, d_hi, d_bad, st));
  int32_t bad = INT_MAX;
  MP_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  if (bad != INT_MAX) {
    // Resolve the reference's first missing endpoint: source, then sinks
    // (plan.cpp:111-116).
    int32_t miss = g->h_edge_src[bad];
    if (timestep_of[miss] != 0) {
      for (int64_t k = g->h_sink_off[bad]; k < g->h_sink_off[bad + 1]; ++k)
        if (timestep_of[g->h_sinks[k]] == 0) {
          miss = g->h_sinks[k];
          break;
        }
    }
    if (missing_node) *missing_node = miss;
    set_error("InvalidOrder: node #" + std::to_string(miss) + " has no timestep");
    return MP_E_INVALID_ORDER;
  }
  if (E) {
    MP_CUDA(cudaMemcpyAsync(lo, d_lo, 4 * E, cudaMemcpyDeviceToHost, st));
    MP_CUDA(cudaMemcpyAsync(hi, d_hi, 4 * E, cudaMemcpyDeviceToHost, st));
    MP_CUDA(cudaStreamSynchronize(st));
  }
  return MP_OK;
}

// ---- resident bytes / timeline ----------------------------------------------------
static mp_status score_one(mp_ctx* ctx, const mp_graph* g, const int32_t* order, int64_t len,
                           uint64_t* bytes, uint64_t* peak) {
  if (!ctx || !g || (len > 0 && !order)) return invalid_arg("null argument");
  if (len != g->n) return invalid_order();
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t n = (size_t)g->n;
  MP_TRY(ctx->scratch[0].reserve(Carver::size_of({4 * n, 8 * n, 8, 4, 1})));
  Carver cv(ctx->scratch[0].ptr);
  int32_t* d_order = cv.take<int32_t>(n);
  uint64_t* d_bytes = cv.take<uint64_t>(n);
  uint64_t* d_peak = cv.take<uint64_t>(1);
  int32_t* d_step = cv.take<int32_t>(1);
  uint8_t* d_valid = cv.take<uint8_t>(1);
  if (n == 0) {
    if (peak) *peak = 0;
    return MP_OK;
  }
  MP_CUDA(cudaMemcpyAsync(d_order, order, 4 * n, cudaMemcpyHostToDevice, st));
  MP_TRY(launch_score(g, d_order, 1, d_peak, d_step, d_valid, bytes ? d_bytes : nullptr,
                       nullptr, 0, st));
  uint8_t valid = 0;
  uint64_t pk = 0;
  MP_CUDA(cudaMemcpyAsync(&valid, d_valid, 1, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaMemcpyAsync(&pk, d_peak, 8, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  if (!valid) return invalid_order();
  if (bytes) {
    MP_CUDA(cudaMemcpyAsync(bytes, d_bytes, 8 * n, cudaMemcpyDeviceToHost, st));
    MP_CUDA(cudaStreamSynchronize(st));
  }
  if (peak) *peak = pk;
  return MP_OK;
}

mp_status mp_resident_bytes(mp_ctx* ctx, const mp_graph* g, const int32_t* order, int64_t len,
                            uint64_t* bytes) {
  MP_TRY(same_ctx(ctx, g));
  if (g && g->n > 0 && !bytes) return invalid_arg("bytes is null");
  return score_one(ctx, g, order, len, bytes, nullptr);
}

mp_status mp_peak_resident_bytes(mp_ctx* ctx, const mp_graph* g, const int32_t* order,
                                 int64_t len, uint64_t* peak) {
  MP_TRY(same_ctx(ctx, g));
  if (!peak) return invalid_arg("peak is null");
  return score_one(ctx, g, order, len, nullptr, peak);
}

mp_status mp_timeline(mp_ctx* ctx, const mp_graph* g, const int32_t* lo, const int32_t* hi,
                      int32_t horizon, uint64_t* bytes, uint64_t* peak_rs, int32_t* peak_step) {
  MP_TRY(same_ctx(ctx, g));
  if (!ctx || !g || (g->E > 0 && (!lo || !hi)) || !peak_rs || !peak_step)
    return invalid_arg("null argument");
  if (horizon < 0) return invalid_arg("negative horizon");
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t E = (size_t)g->E, h = (size_t)horizon;
  MP_TRY(ctx->scratch[0].reserve(Carver::size_of({4 * E, 4 * E, 8 * h, 8 * (h + 2), 8, 4})));
  Carver cv(ctx->scratch[0].ptr);
  int32_t* d_lo = cv.take<int32_t>(E);
  int32_t* d_hi = cv.take<int32_t>(E);
  uint64_t* d_bytes = cv.take<uint64_t>(h);
  int64_t* d_diff = cv.take<int64_t>(h + 2);
  uint64_t* d_peak = cv.take<uint64_t>(1);
  int32_t* d_step = cv.take<int32_t>(1);
  if (E) {
    MP_CUDA(cudaMemcpyAsync(d_lo, lo, 4 * E, cudaMemcpyHostToDevice, st));
    MP_CUDA(cudaMemcpyAsync(d_hi, hi, 4 * E, cudaMemcpyHostToDevice, st));
  }
  MP_TRY(launch_timeline(g->E, d_lo, d_hi, g->d_edge_size, horizon, bytes ? d_bytes : nullptr,
                         d_peak, d_step, d_diff, st));
  MP_CUDA(cudaMemcpyAsync(peak_rs, d_peak, 8, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaMemcpyAsync(peak_step, d_step, 4, cudaMemcpyDeviceToHost, st));
  if (bytes && h) MP_CUDA(cudaMemcpyAsync(bytes, d_bytes, 8 * h, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  return MP_OK;
}

// ---- batched scoring --------------------------------------------------------------
mp_status mp_score_orders_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_orders,
                            int64_t C, uint64_t* d_peak, int32_t* d_step, uint8_t* d_valid,
                            void* stream) {
  return mp_score_orders_argmin_d(ctx, g, d_orders, C, d_peak, d_step, d_valid, nullptr, 0,
                                  stream);
}

mp_status mp_score_orders_argmin_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_orders,
                                   int64_t C, uint64_t* d_peak, int32_t* d_step,
                                   uint8_t* d_valid, uint64_t* d_best_key, int64_t index_base,
                                   void* stream) {
  MP_TRY(same_ctx(ctx, g));
  if (!ctx || !g || C < 0 || index_base < 0) return invalid_arg("null argument or negative count");
  if (C > 0 && (!d_peak || !d_step || !d_valid || (g->n > 0 && !d_orders)))
    return invalid_arg("null output");
  DeviceGuard guard(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL: default stream
  return launch_score(g, d_orders, C, d_peak, d_step, d_valid, nullptr, d_best_key, index_base,
                      st);
}

mp_status mp_score_orders(mp_ctx* ctx, const mp_graph* g, const int32_t* orders, int64_t C,
                          uint64_t* peak, int32_t* step, uint8_t* valid) {
  return mp_score_orders_best(ctx, g, orders, C, peak, step, valid, nullptr);
}

namespace {
// int32 orders -> uint16 (values outside [0, n) become 0xffff, still out of range
// for the kernel since n < 65535), on the host cores: the packed orders halve the
// PCIe bytes of the host-buffer call, the transfer that bounds it.
// int32 orders -> 3-byte ids, little-endian (values outside [0, n) become 0xffffff,
// still out of range since n < 0xffffff): the node-partitioned scorer's wire format.
void pack_orders24(const int32_t* src, uint8_t* dst, size_t cnt, uint32_t n) {
  static const int nthr = [] {
    const char* e = std::getenv("MP_PACK_THREADS");
    const int hw = (int)std::thread::hardware_concurrency();
    const int v = e ? std::atoi(e) : (hw < 16 ? hw : 16);
    return v < 1 ? 1 : v;
  }();
  const int t = cnt < (size_t{1} << 16) ? 1 : nthr;
  const int64_t groups = (int64_t)(cnt / 4);  // n % 4 == 0: rows are whole groups
#pragma omp parallel for num_threads(t) schedule(static)
  for (int64_t q = 0; q < groups; ++q) {
    uint32_t v[4];
    for (int h = 0; h < 4; ++h) {
      const uint32_t x = (uint32_t)src[4 * q + h];
      v[h] = x < n ? x : 0xffffffu;
    }
    uint32_t* w = reinterpret_cast<uint32_t*>(dst + 12 * q);
    w[0] = v[0] | v[1] << 24;
    w[1] = v[1] >> 8 | v[2] << 16;
    w[2] = v[2] >> 16 | v[3] << 8;
  }
}

void pack_orders16(const int32_t* src, uint16_t* dst, size_t cnt, uint32_t n) {
  static const int nthr = [] {
    const char* e = std::getenv("MP_PACK_THREADS");
    const int hw = (int)std::thread::hardware_concurrency();
    const int v = e ? std::atoi(e) : (hw < 16 ? hw : 16);
    return v < 1 ? 1 : v;
  }();
  const int t = cnt < (size_t{1} << 16) ? 1 : nthr;
#pragma omp parallel for num_threads(t) schedule(static)
  for (int64_t i = 0; i < (int64_t)cnt; ++i) {
    const uint32_t v = (uint32_t)src[i];
    dst[i] = v < n ? (uint16_t)v : (uint16_t)0xffffu;
  }
}
}  // namespace

namespace mpb {
// A large device result into caller (typically pageable) memory: chunks land in a
// pinned double buffer at PCIe speed and the host cores copy each one out while
// the next is in flight, instead of the driver's single-threaded pageable staging.
// Synchronises `st`.
mp_status d2h_large(mp_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  constexpr size_t kChunk = size_t{4} << 20;
  if (bytes < 2 * kChunk) {
    MP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    MP_CUDA(cudaStreamSynchronize(st));
    return MP_OK;
  }
  if (!ctx->h_bounce) MP_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_bounce), 2 * kChunk));
  static const int nthr = [] {
    const int hw = (int)std::thread::hardware_concurrency();
    return hw < 1 ? 1 : hw < 16 ? hw : 16;
  }();
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](size_t i) -> mp_status {
    const size_t off = i * kChunk, len = bytes - off < kChunk ? bytes - off : kChunk;
    MP_CUDA(cudaMemcpyAsync(ctx->h_bounce + (i & 1) * kChunk,
                            static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, st));
    MP_CUDA(cudaEventRecord(ctx->ev_d2h[i & 1], st));
    return MP_OK;
  };
  MP_TRY(issue(0));
  for (size_t i = 0; i < nch; ++i) {
    if (i + 1 < nch) MP_TRY(issue(i + 1));  // its half was drained in iteration i - 1
    MP_CUDA(cudaEventSynchronize(ctx->ev_d2h[i & 1]));
    const size_t off = i * kChunk, len = bytes - off < kChunk ? bytes - off : kChunk;
    const char* from = ctx->h_bounce + (i & 1) * kChunk;
    char* to = static_cast<char*>(dst) + off;
    const int64_t parts = nthr;
#pragma omp parallel for num_threads(nthr) schedule(static)
    for (int64_t t = 0; t < parts; ++t) {
      const size_t b = len * (size_t)t / (size_t)parts, e = len * (size_t)(t + 1) / (size_t)parts;
      std::memcpy(to + b, from + b, e - b);
    }
  }
  MP_CUDA(cudaStreamSynchronize(st));
  return MP_OK;
}
}  // namespace mpb

namespace mpb {
// Reduces the fused {key, overflow} pair on the device across shards (NCCL), on
// the scoring stream, before the key is read back. Null: single shard.
struct KeyReduce {
  mp_status (*fn)(void* arg, uint64_t* d_key, cudaStream_t st) = nullptr;
  void* arg = nullptr;
  int64_t index_base = 0;  // global index of this shard's first candidate
};
mp_status score_best_impl(mp_ctx* ctx, const mp_graph* g, const int32_t* orders, int64_t C,
                          uint64_t* peak, int32_t* step, uint8_t* valid, int64_t* best,
                          const KeyReduce* kr, bool* key_overflow);
}  // namespace mpb

mp_status mp_score_orders_best(mp_ctx* ctx, const mp_graph* g, const int32_t* orders, int64_t C,
                               uint64_t* peak, int32_t* step, uint8_t* valid, int64_t* best) {
  return score_best_impl(ctx, g, orders, C, peak, step, valid, best, nullptr, nullptr);
}

mp_status mpb::score_best_impl(mp_ctx* ctx, const mp_graph* g, const int32_t* orders, int64_t C,
                               uint64_t* peak, int32_t* step, uint8_t* valid, int64_t* best,
                               const KeyReduce* kr, bool* key_overflow) {
  if (!ctx || !g || C < 0) return invalid_arg("null argument or negative count");
  if (g->ctx != ctx) return invalid_arg("graph belongs to another context");
  if (best) *best = -1;
  if (key_overflow) *key_overflow = false;
  const int64_t gbase = kr ? kr->index_base : 0;
  if (C == 0 && !kr) return MP_OK;
  if (C > 0 && (!peak || !step || !valid || (g->n > 0 && !orders))) return invalid_arg("null buffer");
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t n = (size_t)g->n, c = (size_t)C;
  MP_TRY(ctx->scratch[0].reserve(Carver::size_of({4 * n * c, 8 * c, 4 * c, c, 24})));
  Carver cv(ctx->scratch[0].ptr);
  int32_t* d_orders = cv.take<int32_t>(n * c);
  uint64_t* d_peak = cv.take<uint64_t>(c);
  int32_t* d_step = cv.take<int32_t>(c);
  uint8_t* d_valid = cv.take<uint8_t>(c);
  uint64_t* d_key = cv.take<uint64_t>(3);
  const bool fused = (best || kr) && gbase + C <= (int64_t{1} << 20);
  uint64_t* hk = ctx->h_small;  // pinned: async copies, no staging
  if (fused) MP_CUDA(cudaMemsetAsync(d_key, 0x7f, 16, st));  // {MP_KEY_NONE, no overflow}
  // Pipeline: the orders go up in chunks on the copy stream while the previous
  // chunk is scored on `st`; each chunk's results come back on `st` (the other
  // copy direction), so only the last chunk's kernel and read-back are exposed.
  // Chunks are >= 4 MiB of orders (at most 4 by default); the per-chunk key accumulates into one
  // first minimum (index_base = chunk offset).
  const size_t bytes = 4 * n * c;
  int64_t nch = (int64_t)(bytes >> 22);
  static const int max_ch = [] {  // MP_PIPE_CHUNKS caps the chunk count (1 = no pipeline)
    const char* e = std::getenv("MP_PIPE_CHUNKS");
    const int v = e ? std::atoi(e) : 4;  // 2-4 measured best at C2/C3 (8 adds launch gaps)
    return v < 1 ? 1 : v > mp_ctx::kPipeChunks ? mp_ctx::kPipeChunks : v;
  }();
  if (nch > max_ch) nch = max_ch;
  if (nch > C) nch = C;
  if (nch < 1 || n == 0) nch = 1;
  // Packed orders on the wire when the graph's scorer takes them: 16-bit for the
  // register-slot variant (n < 65535), 3-byte ids for the node-partitioned one.
  const bool p16 = n > 0 && score_takes_u16(g) && !std::getenv("MP_NO_PACK16");
  // (3-byte ids are opt-in, MP_PACK24=1: on the 16-core host of the measuring box
  // the pack itself bounds the call - 8.6e4 vs 1.0e5 plans/s end to end at C5 - since
  // it reads 4 B and writes 3 B per id to save 1 B of PCIe)
  const bool p24 = !p16 && n > 0 && score_takes_u24(g) && std::getenv("MP_PACK24");
  const size_t wire = p16 ? 2 : p24 ? 3 : 4;  // bytes per id on the wire
  const int ofmt = p16 ? kOrdU16 : p24 ? kOrdU24 : kOrdI32;
  uint8_t* dw = reinterpret_cast<uint8_t*>(d_orders);
  const size_t half = wire * n * (size_t)((C + nch - 1) / nch);  // bytes per staging half
  // a call that failed part-way may have left copies from the staging buffer queued
  if (wire < 4) MP_CUDA(cudaStreamSynchronize(ctx->copy_stream));
  if (wire < 4 && ctx->h_stage_bytes < half) {
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    ctx->h_stage = nullptr;
    ctx->h_stage_bytes = 0;
    MP_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_stage), 2 * half));
    ctx->h_stage_bytes = half;
  }
  cudaStream_t cs = nch > 1 ? ctx->copy_stream : st;
  if (nch > 1) {  // the copy stream starts after everything already queued on `st`
    MP_CUDA(cudaEventRecord(ctx->ev_start, st));
    MP_CUDA(cudaStreamWaitEvent(cs, ctx->ev_start, 0));
  }
  for (int64_t k = 0; k < nch; ++k) {
    const int64_t b = C * k / nch, e = C * (k + 1) / nch, m = e - b;
    if (wire < 4) {  // pack chunk k while chunk k - 1 is on the wire (two staging halves)
      uint8_t* buf = ctx->h_stage + (size_t)(k & 1) * ctx->h_stage_bytes;
      if (k >= 2) MP_CUDA(cudaEventSynchronize(ctx->ev_h2d[k - 2]));  // this half is free
      if (p16)
        pack_orders16(orders + (size_t)b * n, reinterpret_cast<uint16_t*>(buf), n * (size_t)m,
                      (uint32_t)n);
      else
        pack_orders24(orders + (size_t)b * n, buf, n * (size_t)m, (uint32_t)n);
      MP_CUDA(cudaMemcpyAsync(dw + wire * (size_t)b * n, buf, wire * n * (size_t)m,
                              cudaMemcpyHostToDevice, cs));
    } else if (n) {
      MP_CUDA(cudaMemcpyAsync(d_orders + (size_t)b * n, orders + (size_t)b * n,
                              4 * n * (size_t)m, cudaMemcpyHostToDevice, cs));
    }
    if (nch > 1 || wire < 4) {
      MP_CUDA(cudaEventRecord(ctx->ev_h2d[k], cs));
      if (nch > 1) MP_CUDA(cudaStreamWaitEvent(st, ctx->ev_h2d[k], 0));
    }
    const int32_t* chunk = reinterpret_cast<const int32_t*>(dw + wire * (size_t)b * n);
    MP_TRY(launch_score(g, chunk, m, d_peak + b, d_step + b, d_valid + b, nullptr,
                        fused ? d_key : nullptr, gbase + b, st, ofmt));
    MP_CUDA(cudaMemcpyAsync(peak + b, d_peak + b, 8 * (size_t)m, cudaMemcpyDeviceToHost, st));
    MP_CUDA(cudaMemcpyAsync(step + b, d_step + b, 4 * (size_t)m, cudaMemcpyDeviceToHost, st));
    MP_CUDA(cudaMemcpyAsync(valid + b, d_valid + b, (size_t)m, cudaMemcpyDeviceToHost, st));
  }
  if (kr) {  // every shard takes part in the reduction, overflowed or not
    if (!fused) MP_CUDA(cudaMemsetAsync(d_key, 0, 16, st));  // {0, overflow}: forces the fallback
    MP_TRY(kr->fn(kr->arg, d_key, st));
  }
  if (fused || kr) MP_CUDA(cudaMemcpyAsync(hk, d_key, 16, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  if (kr) {  // the reduced pair: global first minimum, or every shard falls back
    if (hk[1] == 0) {
      if (key_overflow) *key_overflow = true;
    } else if (best) {
      *best = hk[0] == MP_KEY_NONE ? -1 : (int64_t)(hk[0] & ((1ull << 20) - 1));
    }
    return MP_OK;
  }
  if (best) {
    if (fused && hk[1] != 0 && hk[0] == MP_KEY_NONE) {
      *best = -1;                                     // no valid candidate
    } else if (fused && hk[1] != 0) {
      *best = (int64_t)(hk[0] & ((1ull << 20) - 1));  // fused (peak, index) minimum
    } else {                                          // a key overflowed: reduce on the device
      MP_TRY(launch_argmin(d_peak, d_valid, C, 0, d_key, st));
      MP_CUDA(cudaMemcpyAsync(hk, d_key, 8, cudaMemcpyDeviceToHost, st));
      MP_CUDA(cudaStreamSynchronize(st));
      *best = (int64_t)hk[0];
    }
  }
  return MP_OK;
}

mp_status mp_key_reset_d(mp_ctx* ctx, uint64_t* d_best_key, void* stream) {
  if (!ctx || !d_best_key) return invalid_arg("null argument");
  DeviceGuard guard(ctx->device);
  MP_CUDA(cudaMemsetAsync(d_best_key, 0x7f, 16, static_cast<cudaStream_t>(stream)));
  return MP_OK;
}

mp_status mp_argmin_key_d(mp_ctx* ctx, const uint64_t* d_peak, const uint8_t* d_valid,
                          int64_t C, int64_t index_base, uint64_t* d_out3, void* stream) {
  if (!ctx || !d_out3 || C < 0 || index_base < 0 || (C > 0 && (!d_peak || !d_valid)))
    return invalid_arg("bad argument");
  DeviceGuard guard(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL: default stream
  return launch_argmin(d_peak, d_valid, C, index_base, d_out3, st);
}

mp_status mp_argmin(mp_ctx* ctx, const uint64_t* peak, const uint8_t* valid, int64_t C,
                    int64_t* best) {
  if (!ctx || !best || C < 0 || (C > 0 && (!peak || !valid))) return invalid_arg("bad argument");
  *best = -1;
  if (C == 0) return MP_OK;
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t c = (size_t)C;
  MP_TRY(ctx->scratch[1].reserve(Carver::size_of({8 * c, c, 24})));
  Carver cv(ctx->scratch[1].ptr);
  uint64_t* d_peak = cv.take<uint64_t>(c);
  uint8_t* d_valid = cv.take<uint8_t>(c);
  uint64_t* d_out = cv.take<uint64_t>(3);
  MP_CUDA(cudaMemcpyAsync(d_peak, peak, 8 * c, cudaMemcpyHostToDevice, st));
  MP_CUDA(cudaMemcpyAsync(d_valid, valid, c, cudaMemcpyHostToDevice, st));
  MP_TRY(launch_argmin(d_peak, d_valid, C, 0, d_out, st));
  uint64_t out[3];
  MP_CUDA(cudaMemcpyAsync(out, d_out, 24, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  *best = (int64_t)out[0];
  return MP_OK;
}

// ---- overlap pairs / validation ------------------------------------------------------
static mp_status pair_sweep_d(mp_ctx* ctx, PairArgs a, int64_t* d_row_off, int32_t* d_out,
                              int64_t cap, int64_t* count, cudaStream_t st) {
  if (a.row_begin < 0 || a.row_end < a.row_begin || a.row_end > a.num_edges)
    return invalid_arg("row range out of bounds");
  MP_TRY(ctx->scratch[2].reserve(pairs_scratch_bytes(a, ctx->num_sms)));
  int64_t total = 0;
  if (!d_out || cap <= 0) {
    MP_TRY(pairs_count(a, ctx->num_sms, ctx->scratch[2].ptr, d_row_off, &total, st));
    *count = total;
    if (d_out && total > 0) {
      set_error("Capacity: " + std::to_string(total) + " pairs exceed the buffer of 0");
      return MP_E_CAPACITY;
    }
    return MP_OK;
  }
  // count -> scan -> fill back to back (the fill writes at most `cap` pairs), one
  // read-back of the total at the end
  MP_TRY(pairs_count(a, ctx->num_sms, ctx->scratch[2].ptr, d_row_off, nullptr, st));
  MP_TRY(pairs_fill(a, ctx->num_sms, ctx->scratch[2].ptr, d_row_off, d_out, st, cap));
  MP_CUDA(cudaMemcpyAsync(&total, pairs_device_total(a, ctx->num_sms, ctx->scratch[2].ptr),
                          sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  *count = total;
  if (total > cap) {
    set_error("Capacity: " + std::to_string(total) + " pairs exceed the buffer of " +
              std::to_string(cap) + " (the first " + std::to_string(cap) + " were written)");
    return MP_E_CAPACITY;
  }
  return MP_OK;
}

static mp_status pair_sweep_h(mp_ctx* ctx, int mode, int32_t E, const int32_t* lo,
                              const int32_t* hi, const uint64_t* size, const uint8_t* mask,
                              const uint64_t* addr, int32_t* out, int64_t cap, int64_t* count) {
  if (!ctx || !count || E < 0 || (E > 0 && (!lo || !hi || !size)))
    return invalid_arg("null argument");
  if (mode == 1 && E > 0 && (!mask || !addr)) return invalid_arg("null address arrays");
  *count = 0;
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t e = (size_t)E;
  MP_TRY(ctx->scratch[0].reserve(Carver::size_of({4 * e, 4 * e, 8 * e, e, 8 * e, 8 * (e + 1)})));
  Carver cv(ctx->scratch[0].ptr);
  int32_t* d_lo = cv.take<int32_t>(e);
  int32_t* d_hi = cv.take<int32_t>(e);
  uint64_t* d_size = cv.take<uint64_t>(e);
  uint8_t* d_mask = cv.take<uint8_t>(e);
  uint64_t* d_addr = cv.take<uint64_t>(e);
  int64_t* d_row_off = cv.take<int64_t>(e + 1);
  if (E == 0) return MP_OK;
  MP_CUDA(cudaMemcpyAsync(d_lo, lo, 4 * e, cudaMemcpyHostToDevice, st));
  MP_CUDA(cudaMemcpyAsync(d_hi, hi, 4 * e, cudaMemcpyHostToDevice, st));
  MP_CUDA(cudaMemcpyAsync(d_size, size, 8 * e, cudaMemcpyHostToDevice, st));
  if (mask) MP_CUDA(cudaMemcpyAsync(d_mask, mask, e, cudaMemcpyHostToDevice, st));
  if (addr) MP_CUDA(cudaMemcpyAsync(d_addr, addr, 8 * e, cudaMemcpyHostToDevice, st));
  PairArgs a;
  a.num_edges = E;
  a.lo = d_lo;
  a.hi = d_hi;
  a.size = d_size;
  a.mask = mask ? d_mask : nullptr;
  a.addr = addr ? d_addr : nullptr;
  a.mode = mode;
  a.row_begin = 0;
  a.row_end = E;
  int64_t total = 0;
  MP_TRY(ctx->scratch[2].reserve(pairs_scratch_bytes(a, ctx->num_sms)));
  MP_TRY(pairs_count(a, ctx->num_sms, ctx->scratch[2].ptr, d_row_off, &total, st));
  *count = total;
  if (!out) return MP_OK;
  if (total > cap) {
    set_error("Capacity: " + std::to_string(total) + " pairs exceed the buffer of " +
              std::to_string(cap));
    return MP_E_CAPACITY;
  }
  if (total == 0) return MP_OK;
  MP_TRY(ctx->scratch[1].reserve((size_t)total * 8 + 256));
  int32_t* d_out = static_cast<int32_t*>(ctx->scratch[1].ptr);
  MP_TRY(pairs_fill(a, ctx->num_sms, ctx->scratch[2].ptr, d_row_off, d_out, st));
  return d2h_large(ctx, out, d_out, (size_t)total * 8, st);
}

mp_status mp_overlap_pairs(mp_ctx* ctx, int32_t E, const int32_t* lo, const int32_t* hi,
                           const uint64_t* size, const uint8_t* pinned, int32_t* pairs,
                           int64_t cap, int64_t* count) {
  return pair_sweep_h(ctx, 0, E, lo, hi, size, pinned, nullptr, pairs, cap, count);
}

mp_status mp_overlap_pairs_d(mp_ctx* ctx, int32_t E, const int32_t* d_lo, const int32_t* d_hi,
                             const uint64_t* d_size, const uint8_t* d_pinned, int64_t row_begin,
                             int64_t row_end, int64_t* d_row_off, int32_t* d_pairs, int64_t cap,
                             int64_t* count, void* stream) {
  if (!ctx || !count || !d_row_off || E < 0 || (E > 0 && (!d_lo || !d_hi || !d_size)))
    return invalid_arg("null argument");
  DeviceGuard guard(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL: default stream
  PairArgs a;
  a.num_edges = E;
  a.lo = d_lo;
  a.hi = d_hi;
  a.size = d_size;
  a.mask = d_pinned;
  a.mode = 0;
  a.row_begin = row_begin;
  a.row_end = row_end;
  return pair_sweep_d(ctx, a, d_row_off, d_pairs, cap, count, st);
}

mp_status mp_validate_pairs(mp_ctx* ctx, int32_t E, const int32_t* lo, const int32_t* hi,
                            const uint64_t* size, const uint8_t* has_addr, const uint64_t* addr,
                            int32_t* viol, int64_t cap, int64_t* num_viol) {
  return pair_sweep_h(ctx, 1, E, lo, hi, size, has_addr, addr, viol, cap, num_viol);
}

mp_status mp_validate_pairs_d(mp_ctx* ctx, int32_t E, const int32_t* d_lo, const int32_t* d_hi,
                              const uint64_t* d_size, const uint8_t* d_has, const uint64_t* d_addr,
                              int64_t row_begin, int64_t row_end, int64_t* d_row_off,
                              int32_t* d_viol, int64_t cap, int64_t* num_viol, void* stream) {
  if (!ctx || !num_viol || !d_row_off || E < 0 ||
      (E > 0 && (!d_lo || !d_hi || !d_size || !d_has || !d_addr)))
    return invalid_arg("null argument");
  DeviceGuard guard(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL: default stream
  PairArgs a;
  a.num_edges = E;
  a.lo = d_lo;
  a.hi = d_hi;
  a.size = d_size;
  a.mask = d_has;
  a.addr = d_addr;
  a.mode = 1;
  a.row_begin = row_begin;
  a.row_end = row_end;
  return pair_sweep_d(ctx, a, d_row_off, d_viol, cap, num_viol, st);
}

// ---- one process, several GPUs (§8e) ------------------------------------------------
// NCCL is loaded at run time (the library does not link it, so a process without
// NCCL still scores on one GPU); its few entry points are resolved by name.
namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    if (std::getenv("MP_NO_NCCL")) {
      a.why = "MP_NO_NCCL set";
      return a;
    }
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = "libnccl.so.2 not found";
      return a;
    }
    a.comm_init_all = reinterpret_cast<decltype(a.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.comm_init_all && a.all_reduce && a.comm_destroy && a.error_string;
    if (!a.ok) a.why = "libnccl lacks ncclCommInitAll/ncclAllReduce";
    return a;
  }();
  return api;
}

// one shard's part of the single allreduce(MIN) over the 16-byte {key, overflow}
mp_status nccl_min_key(void* comm, uint64_t* d_key, cudaStream_t st) {
  const ncclResult_t r = nccl().all_reduce(d_key, d_key, 2, ncclInt64, ncclMin,
                                           static_cast<ncclComm_t>(comm), st);
  if (r != ncclSuccess) {
    set_error(std::string("ncclAllReduce: ") + nccl().error_string(r));
    return MP_E_CUDA;
  }
  return MP_OK;
}
}  // namespace

mp_status mp_multi_create(const int* devices, int G, mp_multi** out) {
  if (!devices || G <= 0 || !out) return invalid_arg("null argument or no devices");
  *out = nullptr;
  auto* m = new mp_multi();
  for (int i = 0; i < G; ++i) {
    mp_ctx* c = nullptr;
    const mp_status s = mp_ctx_create(devices[i], &c);
    if (s != MP_OK) {
      mp_multi_destroy(m);
      return s;
    }
    m->ctx.push_back(c);
  }
  // one communicator per device when the devices are distinct (NCCL cannot put
  // two ranks of one communicator on one GPU); otherwise the host combine
  std::vector<int> devs(devices, devices + G);
  std::vector<int> sorted = devs;
  std::sort(sorted.begin(), sorted.end());
  if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end()) {
    m->nccl_note = "repeated device entries";
  } else if (!nccl().ok) {
    m->nccl_note = nccl().why;
  } else {
    std::vector<ncclComm_t> comms(G);
    const ncclResult_t r = nccl().comm_init_all(comms.data(), G, devs.data());
    if (r == ncclSuccess) {
      m->comm.assign(comms.begin(), comms.end());
    } else {
      m->nccl_note = std::string("ncclCommInitAll: ") + nccl().error_string(r);
    }
  }
  *out = m;
  return MP_OK;
}

mp_status mp_multi_destroy(mp_multi* m) {
  if (!m) return MP_OK;
  for (void* c : m->comm) nccl().comm_destroy(static_cast<ncclComm_t>(c));
  for (mp_graph* g : m->graph) mp_graph_free(g);
  for (mp_ctx* c : m->ctx) mp_ctx_destroy(c);
  delete m;
  return MP_OK;
}

int mp_multi_nccl(const mp_multi* m) { return m && !m->comm.empty() ? 1 : 0; }

mp_status mp_multi_upload(mp_multi* m, const mp_csr* csr) {
  if (!m || !csr) return invalid_arg("null argument");
  for (mp_graph* g : m->graph) mp_graph_free(g);
  m->graph.assign(m->ctx.size(), nullptr);
  for (size_t i = 0; i < m->ctx.size(); ++i) MP_TRY(mp_graph_upload(m->ctx[i], csr, &m->graph[i]));
  return MP_OK;
}

mp_status mp_score_orders_multi(mp_multi* m, const int32_t* orders, int64_t C, uint64_t* peak,
                                int32_t* step, uint8_t* valid, int64_t* best) {
  if (!m || C < 0 || m->graph.empty() || !m->graph[0]) return invalid_arg("no graph uploaded");
  if (best) *best = -1;
  if (C == 0) return MP_OK;
  const int G = (int)m->ctx.size();
  const int64_t n = m->graph[0]->n;
  const bool use_nccl = !m->comm.empty();
  std::vector<mp_status> st(G, MP_OK);
  std::vector<std::string> err(G);
  std::vector<int64_t> lbest(G, -1), gbest(G, -1), beg(G + 1);
  std::vector<char> over(G, 0);
  for (int i = 0; i <= G; ++i) beg[i] = C * i / G;  // contiguous shards, as shard_range
  std::vector<std::thread> pool;
  for (int i = 0; i < G; ++i)
    pool.emplace_back([&, i] {
      const int64_t b = beg[i], c = beg[i + 1] - beg[i];
      KeyReduce kr;
      kr.fn = [](void* comm, uint64_t* d_key, cudaStream_t s) { return nccl_min_key(comm, d_key, s); };
      kr.arg = use_nccl ? m->comm[i] : nullptr;
      kr.index_base = b;
      bool ovf = false;
      // NCCL: every shard's fused key goes through ONE allreduce(MIN) on the device
      // and each thread reads back the global first minimum; otherwise each shard's
      // own first minimum comes back and the host combines them.
      st[i] = score_best_impl(m->ctx[i], m->graph[i], orders ? orders + b * n : nullptr, c,
                              peak + b, step + b, valid + b, use_nccl ? &gbest[i] : &lbest[i],
                              use_nccl ? &kr : nullptr, &ovf);
      over[i] = ovf ? 1 : 0;
      if (st[i] != MP_OK) err[i] = mp_last_error();
    });
  for (std::thread& t : pool) t.join();
  for (int i = 0; i < G; ++i)
    if (st[i] != MP_OK) {
      set_error(err[i]);
      return st[i];
    }
  if (use_nccl && !over[0]) {  // the reduced key is the same on every device
    if (best) *best = gbest[0];
    return MP_OK;
  }
  // host combine: first minimum over the scores, in index order (also the NCCL
  // path's fallback when some shard's key did not fit)
  int64_t bi = -1;
  if (use_nccl) {
    for (int64_t c = 0; c < C; ++c)
      if (valid[c] && (bi < 0 || peak[c] < peak[bi])) bi = c;
  } else {
    for (int i = 0; i < G; ++i) {
      if (lbest[i] < 0) continue;
      const int64_t gi = beg[i] + lbest[i];
      if (bi < 0 || peak[gi] < peak[bi]) bi = gi;
    }
  }
  if (best) *best = bi;
  return MP_OK;
}

// ---- joint-mode pair set (K8) -----------------------------------------------------
namespace {
// compute_levels / compute_bounds (analysis.cpp:11-62) and the AR bitsets of k_joint.cu
mp_status joint_tables(mp_graph* g) {
  if (g->d_joint_mul) return MP_OK;
  const int32_t n = g->n, E = g->E;
  const size_t Wn = ((size_t)n + 31) / 32, WEn = ((size_t)E + 31) / 32;
  const size_t host_bytes = 4 * Wn * ((size_t)n + (size_t)E);   // desc + AR
  const size_t dev_bytes = 4 * (Wn * (size_t)E + WEn * (size_t)n);  // AR + ARt
  if (n > kJointMaxNodes || host_bytes > kJointMaxTableBytes || dev_bytes > kJointMaxTableBytes) {
    set_error("Capacity: the joint-mode pair tables support up to " +
              std::to_string(kJointMaxNodes) + " nodes and " +
              std::to_string(kJointMaxTableBytes >> 30) + " GiB of bitsets");
    return MP_E_CAPACITY;
  }
  std::vector<std::vector<int32_t>> succ(n);
  std::vector<int32_t> indeg(n, 0);
  for (int32_t e = 0; e < E; ++e)
    for (int64_t k = g->h_sink_off[e]; k < g->h_sink_off[e + 1]; ++k) {
      succ[g->h_edge_src[e]].push_back(g->h_sinks[k]);
      ++indeg[g->h_sinks[k]];
    }
  std::vector<int32_t> order;
  order.reserve(n);
  for (int32_t v = 0; v < n; ++v)
    if (!indeg[v]) order.push_back(v);
  for (size_t i = 0; i < order.size(); ++i)
    for (int32_t w : succ[order[i]])
      if (--indeg[w] == 0) order.push_back(w);
  if ((int32_t)order.size() != n) {
    set_error("InvalidStructure: graph has a cycle");
    return MP_E_BAD_GRAPH;
  }
  std::vector<int32_t> fwd(n, 0), bwd(n, 0);
  for (int32_t v : order)
    for (int32_t w : succ[v]) fwd[w] = std::max(fwd[w], fwd[v] + 1);
  for (auto it = order.rbegin(); it != order.rend(); ++it)
    for (int32_t w : succ[*it]) bwd[*it] = std::max(bwd[*it], bwd[w] + 1);
  std::vector<int32_t> mul(2 * (size_t)E);
  for (int32_t e = 0; e < E; ++e) {
    const int64_t a = g->h_sink_off[e], b = g->h_sink_off[e + 1];
    int32_t hi = n;
    if (b > a) {
      hi = 0;
      for (int64_t k = a; k < b; ++k) hi = std::max(hi, n - bwd[g->h_sinks[k]]);  // alap
    }
    mul[2 * e] = 1 + fwd[g->h_edge_src[e]];  // asap[src]
    mul[2 * e + 1] = hi;
  }
  const int W = (n + 31) / 32, WE = (E + 31) / 32;
  std::vector<uint32_t> desc((size_t)n * W, 0);  // proper descendants (ReachabilityCache)
  for (auto it = order.rbegin(); it != order.rend(); ++it) {
    uint32_t* dv = &desc[(size_t)*it * W];
    for (int32_t w : succ[*it]) {
      const uint32_t* dw = &desc[(size_t)w * W];
      for (int q = 0; q < W; ++q) dv[q] |= dw[q];
      dv[w >> 5] |= 1u << (w & 31);
    }
  }
  std::vector<uint32_t> ar((size_t)E * W, 0);  // the transpose ARt is built on the device
#pragma omp parallel for schedule(dynamic, 64)
  for (int32_t e = 0; e < E; ++e) {
    const int64_t a = g->h_sink_off[e], b = g->h_sink_off[e + 1];
    if (b == a) continue;  // no sinks: edge_precedes(e, .) needs the window test alone
    uint32_t* r = &ar[(size_t)e * W];
    std::copy(&desc[(size_t)g->h_sinks[a] * W], &desc[(size_t)g->h_sinks[a] * W] + W, r);
    for (int64_t k = a + 1; k < b; ++k) {
      const uint32_t* d = &desc[(size_t)g->h_sinks[k] * W];
      for (int q = 0; q < W; ++q) r[q] &= d[q];
    }
  }
  std::vector<uint32_t>().swap(desc);
  cudaStream_t st = g->ctx->stream;
  mp_status s = MP_OK;
  auto up = [&](mp_status r) {
    if (s == MP_OK) s = r;
  };
  int32_t* d_mul = nullptr;
  up(upload(&d_mul, mul.data(), mul.size(), st));
  up(upload(&g->d_joint_ar, ar.data(), ar.size(), st));
  if (s == MP_OK) {
    void* d_art = nullptr;
    const cudaError_t ce = cudaMalloc(&d_art, 4 * (size_t)n * WE);
    if (ce != cudaSuccess) {
      s = cuda_status(ce, "joint tables (ARt)");
    } else {
      g->d_joint_art = static_cast<uint32_t*>(d_art);
      up(launch_joint_transpose(g->d_joint_ar, E, n, W, WE, g->d_joint_art, st));
    }
  }
  g->d_joint_mul = reinterpret_cast<int2*>(d_mul);
  g->joint_ar_words = W;
  g->joint_art_words = WE;
  if (s == MP_OK) {
    cudaError_t ce = cudaStreamSynchronize(st);  // host tables go out of scope
    if (ce != cudaSuccess) s = cuda_status(ce, "joint tables");
  }
  return s;
}
}  // namespace

mp_status mp_joint_pairs(mp_ctx* ctx, const mp_graph* g, int filter, int32_t* pairs, int64_t cap,
                         int64_t* count) {
  MP_TRY(same_ctx(ctx, g));
  if (!ctx || !g || !count) return invalid_arg("null argument");
  *count = 0;
  DeviceGuard guard(ctx->device);
  mp_graph* mg = const_cast<mp_graph*>(g);  // lazily built tables (graph stays immutable)
  if (g->E == 0) return MP_OK;
  if (filter) MP_TRY(joint_tables(mg));
  cudaStream_t st = ctx->stream;
  const size_t E = (size_t)g->E;
  MP_TRY(ctx->scratch[0].reserve(Carver::size_of({8 * E, 8 * E, lp_scan_scratch(g->E), 8})));
  Carver cv(ctx->scratch[0].ptr);
  int64_t* d_cnt = cv.take<int64_t>(E);
  int64_t* d_off = cv.take<int64_t>(E);
  int64_t* d_sums = reinterpret_cast<int64_t*>(cv.take<char>(lp_scan_scratch(g->E)));
  int64_t* d_tot = cv.take<int64_t>(1);
  JointArgs a;
  a.E = g->E;
  a.filter = filter ? 1 : 0;
  a.size = g->d_edge_size;
  a.src = g->d_edge_src;
  a.mul = g->d_joint_mul;
  a.ar = g->d_joint_ar;
  a.art = g->d_joint_art;
  a.ar_words = g->joint_ar_words;
  a.art_words = g->joint_art_words;
  MP_TRY(launch_joint(a, ctx->num_sms, d_cnt, nullptr, nullptr, st));
  MP_TRY(scan_exclusive_i64(d_cnt, g->E, d_off, d_sums, d_tot, st));
  int64_t total = 0;
  MP_CUDA(cudaMemcpyAsync(&total, d_tot, 8, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  *count = total;
  if (!pairs) return MP_OK;
  if (total > cap) {
    set_error("Capacity: " + std::to_string(total) + " pairs exceed the buffer of " +
              std::to_string(cap));
    return MP_E_CAPACITY;
  }
  if (total == 0) return MP_OK;
  MP_TRY(ctx->scratch[4].reserve(8 * (size_t)total + 256));
  int2* d_pairs = static_cast<int2*>(ctx->scratch[4].ptr);
  MP_TRY(launch_joint(a, ctx->num_sms, nullptr, d_off, d_pairs, st));
  return d2h_large(ctx, pairs, d_pairs, 8 * (size_t)total, st);
}

// ---- LP row emission (K7) ---------------------------------------------------------
namespace {
// lp_format.cpp:30-36: every non-alphanumeric byte becomes '_'
std::string lp_sanitize(const char* s, size_t n) {
  std::string out(s, n);
  for (char& c : out)
    if (!std::isalnum(static_cast<unsigned char>(c))) c = '_';
  return out;
}

// lp_names (lp_format.cpp:75-86) suffixes duplicate sanitized names; this path
// supports graphs whose names need no suffix and says so otherwise.
bool lp_names_unique(const std::vector<std::string>& data_ids) {
  std::unordered_set<std::string> d(data_ids.begin(), data_ids.end());
  if (d.size() != data_ids.size()) return false;  // two ids, one sanitized name
  // below_<A>_<B>_ == below_<A'>_<B'>_ needs A' = A_X and B = X_B' with A, B' ids
  std::unordered_set<std::string> xs;
  for (const std::string& a2 : data_ids)
    for (size_t p = 0; p < a2.size(); ++p)
      if (a2[p] == '_' && d.count(a2.substr(0, p))) xs.insert(a2.substr(p + 1));
  if (xs.empty()) return true;
  for (const std::string& b : data_ids)
    for (size_t q = 0; q < b.size(); ++q)
      if (b[q] == '_' && xs.count(b.substr(0, q)) && d.count(b.substr(q + 1))) return false;
  return true;
}
}  // namespace

mp_status mp_encode_addresses_lp(mp_ctx* ctx, int32_t E, const int32_t* lo, const int32_t* hi,
                                 const uint64_t* size, const uint8_t* pinned,
                                 const uint64_t* pinned_addr, const char* ids,
                                 const int64_t* id_off, char* out, int64_t cap, int64_t* len,
                                 int64_t* counts) {
  if (!ctx || !len || E < 0 || (E > 0 && (!lo || !hi || !size || !ids || !id_off)))
    return invalid_arg("null argument");
  if (pinned && !pinned_addr) return invalid_arg("pinned without pinned_addr");
  *len = 0;
  // names, M and the host-side sections (O(E))
  std::vector<std::string> sid(E);
  std::vector<std::string> data_ids;
  std::string names;
  std::vector<int64_t> name_off(E + 1, 0);
  long long M = 0;
  for (int32_t e = 0; e < E; ++e) {
    sid[e] = lp_sanitize(ids + id_off[e], (size_t)(id_off[e + 1] - id_off[e]));
    names += sid[e];
    name_off[e + 1] = (int64_t)names.size();
    M += (long long)size[e];  // Graph::total_bytes (encode.cpp:325)
    if (size[e] > 0) data_ids.push_back(sid[e]);
  }
  if (!lp_names_unique(data_ids)) {
    set_error("InvalidArgument: edge ids are ambiguous once sanitized for LP "
              "(lp_format.cpp:75-86 would suffix them); not supported by this path");
    return MP_E_INVALID_ARG;
  }
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t e = (size_t)E;
  MP_TRY(ctx->scratch[0].reserve(Carver::size_of(
      {4 * e, 4 * e, 8 * e, e, 8 * e, 8 * (e + 1), names.size() + 1, 8 * (e + 1), 8 * 4})));
  Carver cv(ctx->scratch[0].ptr);
  int32_t* d_lo = cv.take<int32_t>(e);
  int32_t* d_hi = cv.take<int32_t>(e);
  uint64_t* d_size = cv.take<uint64_t>(e);
  uint8_t* d_pin = cv.take<uint8_t>(e);
  uint64_t* d_paddr = cv.take<uint64_t>(e);
  int64_t* d_row_off = cv.take<int64_t>(e + 1);
  char* d_names = cv.take<char>(names.size() + 1);
  int64_t* d_name_off = cv.take<int64_t>(e + 1);
  int64_t* d_tot = cv.take<int64_t>(4);
  int64_t P = 0;
  int32_t* d_pairs = nullptr;
  if (E > 0) {
    MP_CUDA(cudaMemcpyAsync(d_lo, lo, 4 * e, cudaMemcpyHostToDevice, st));
    MP_CUDA(cudaMemcpyAsync(d_hi, hi, 4 * e, cudaMemcpyHostToDevice, st));
    MP_CUDA(cudaMemcpyAsync(d_size, size, 8 * e, cudaMemcpyHostToDevice, st));
    if (pinned) {
      MP_CUDA(cudaMemcpyAsync(d_pin, pinned, e, cudaMemcpyHostToDevice, st));
      MP_CUDA(cudaMemcpyAsync(d_paddr, pinned_addr, 8 * e, cudaMemcpyHostToDevice, st));
    }
    if (!names.empty())
      MP_CUDA(cudaMemcpyAsync(d_names, names.data(), names.size(), cudaMemcpyHostToDevice, st));
    MP_CUDA(cudaMemcpyAsync(d_name_off, name_off.data(), 8 * (e + 1), cudaMemcpyHostToDevice,
                            st));
    // the pair list (K2): encode.cpp:347-357 in (i, j) order
    PairArgs pa;
    pa.num_edges = E;
    pa.lo = d_lo;
    pa.hi = d_hi;
    pa.size = d_size;
    pa.mask = pinned ? d_pin : nullptr;
    pa.mode = 0;
    pa.row_begin = 0;
    pa.row_end = E;
    MP_TRY(ctx->scratch[2].reserve(pairs_scratch_bytes(pa, ctx->num_sms)));
    MP_TRY(pairs_count(pa, ctx->num_sms, ctx->scratch[2].ptr, d_row_off, &P, st));
    if (P > 0) {
      MP_TRY(ctx->scratch[4].reserve(Carver::size_of(
          {8 * (size_t)P, 8 * (size_t)P, 8 * (size_t)P, 8 * (size_t)P, 8 * (size_t)P,
           lp_scan_scratch(P)})));
      Carver c4(ctx->scratch[4].ptr);
      d_pairs = c4.take<int32_t>(2 * (size_t)P);
      int64_t* d_rl = c4.take<int64_t>((size_t)P);
      int64_t* d_bl = c4.take<int64_t>((size_t)P);
      int64_t* d_ro = c4.take<int64_t>((size_t)P);
      int64_t* d_bo = c4.take<int64_t>((size_t)P);
      int64_t* d_sums = reinterpret_cast<int64_t*>(c4.take<char>(lp_scan_scratch(P)));
      MP_TRY(pairs_fill(pa, ctx->num_sms, ctx->scratch[2].ptr, d_row_off, d_pairs, st));
      LpArgs la;
      la.E = E;
      la.P = P;
      la.pairs = reinterpret_cast<const int2*>(d_pairs);
      la.size = d_size;
      la.pinned = pinned ? d_pin : nullptr;
      la.pinned_addr = pinned ? d_paddr : nullptr;
      la.names = d_names;
      la.name_off = d_name_off;
      la.M = M;
      la.row_len = d_rl;
      la.bin_len = d_bl;
      la.row_off = d_ro;
      la.bin_off = d_bo;
      MP_TRY(launch_lp_len(la, ctx->num_sms, st));
      MP_TRY(scan_exclusive_i64(d_rl, P, d_ro, d_sums, d_tot, st));
      MP_TRY(scan_exclusive_i64(d_bl, P, d_bo, d_sums, d_tot + 1, st));
      int64_t tot[2];
      MP_CUDA(cudaMemcpyAsync(tot, d_tot, 16, cudaMemcpyDeviceToHost, st));
      MP_CUDA(cudaStreamSynchronize(st));
      // host sections (O(E)) and the total length
      std::string head = "Minimize\n obj: peak_mem\nSubject To\n";
      std::string peak, bounds = "Bounds\n 0 <= peak_mem <= " + std::to_string(M) + "\n",
                        gens = "Generals\n peak_mem\n";
      int64_t q = 0;
      for (int32_t x = 0; x < E; ++x) {
        if (size[x] == 0) continue;
        const bool pin = pinned && pinned[x];
        const long long v = pin ? (long long)pinned_addr[x] : 0;
        peak += " c" + std::to_string(3 * P + q) + "_peak_address:";
        if (!pin) peak += " +1 addr_" + sid[x] + "_";
        peak += " -1 peak_mem <= " + std::to_string(-(long long)size[x] - v) + "\n";
        if (!pin) {
          bounds += " 0 <= addr_" + sid[x] + "_ <= " + std::to_string(M) + "\n";
          gens += " addr_" + sid[x] + "_\n";
        }
        ++q;
      }
      const std::string bin_head = "Binaries\n", end = "End\n";
      const int64_t o_rows = (int64_t)head.size();
      const int64_t o_peak = o_rows + tot[0];
      const int64_t o_bounds = o_peak + (int64_t)peak.size();
      const int64_t o_gens = o_bounds + (int64_t)bounds.size();
      const int64_t o_binh = o_gens + (int64_t)gens.size();
      const int64_t o_bins = o_binh + (int64_t)bin_head.size();
      const int64_t o_end = o_bins + tot[1];
      *len = o_end + (int64_t)end.size();
      if (counts) {
        counts[0] = counts[1] = counts[2] = P;
        counts[3] = q;
      }
      if (!out) return MP_OK;
      if (*len > cap) {
        set_error("Capacity: the LP text of " + std::to_string(*len) +
                  " bytes exceeds the buffer of " + std::to_string(cap));
        return MP_E_CAPACITY;
      }
      MP_TRY(ctx->scratch[5].reserve((size_t)(tot[0] + tot[1]) + 16));
      char* d_text = static_cast<char*>(ctx->scratch[5].ptr);
      MP_TRY(launch_lp_write(la, d_text, d_text + tot[0], ctx->num_sms, st));
      MP_CUDA(cudaMemcpyAsync(out + o_rows, d_text, (size_t)tot[0], cudaMemcpyDeviceToHost, st));
      MP_CUDA(cudaMemcpyAsync(out + o_bins, d_text + tot[0], (size_t)tot[1],
                              cudaMemcpyDeviceToHost, st));
      std::memcpy(out, head.data(), head.size());
      std::memcpy(out + o_peak, peak.data(), peak.size());
      std::memcpy(out + o_bounds, bounds.data(), bounds.size());
      std::memcpy(out + o_gens, gens.data(), gens.size());
      std::memcpy(out + o_binh, bin_head.data(), bin_head.size());
      std::memcpy(out + o_end, end.data(), end.size());
      MP_CUDA(cudaStreamSynchronize(st));
      return MP_OK;
    }
  }
  // no overlapping pairs: every section is host-sized (O(E))
  std::string text = "Minimize\n obj: peak_mem\nSubject To\n";
  std::string bounds = "Bounds\n 0 <= peak_mem <= " + std::to_string(M) + "\n",
              gens = "Generals\n peak_mem\n";
  int64_t q = 0;
  for (int32_t x = 0; x < E; ++x) {
    if (size[x] == 0) continue;
    const bool pin = pinned && pinned[x];
    const long long v = pin ? (long long)pinned_addr[x] : 0;
    text += " c" + std::to_string(q) + "_peak_address:";
    if (!pin) text += " +1 addr_" + sid[x] + "_";
    text += " -1 peak_mem <= " + std::to_string(-(long long)size[x] - v) + "\n";
    if (!pin) {
      bounds += " 0 <= addr_" + sid[x] + "_ <= " + std::to_string(M) + "\n";
      gens += " addr_" + sid[x] + "_\n";
    }
    ++q;
  }
  text += bounds + gens + "Binaries\nEnd\n";
  *len = (int64_t)text.size();
  if (counts) {
    counts[0] = counts[1] = counts[2] = 0;
    counts[3] = q;
  }
  if (!out) return MP_OK;
  if (*len > cap) {
    set_error("Capacity: the LP text of " + std::to_string(*len) + " bytes exceeds the buffer of " +
              std::to_string(cap));
    return MP_E_CAPACITY;
  }
  std::memcpy(out, text.data(), text.size());
  return MP_OK;
}

// ---- arena baseline (K6) -----------------------------------------------------------
mp_status mp_run_baseline_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_orders, int64_t B,
                            int best_fit, uint64_t* d_mr, uint64_t* d_rs, double* d_frag,
                            uint8_t* d_valid, void* stream) {
  MP_TRY(same_ctx(ctx, g));
  if (!ctx || !g || B < 0) return invalid_arg("null argument");
  if (B == 0) return MP_OK;
  if ((!d_orders && g->n > 0) || !d_mr || !d_rs || !d_frag || !d_valid)
    return invalid_arg("null argument");
  ArenaArgs a;
  a.n = g->n;
  a.E = g->E;
  if (arena_smem_bytes(g->n, g->E, 2 * g->E + 2, 8, 0) > (size_t)ctx->max_smem_optin) {
    set_error("Capacity: run_baseline state for " + std::to_string(g->n) + " nodes / " +
              std::to_string(g->E) + " edges exceeds shared memory");
    return MP_E_CAPACITY;
  }
  DeviceGuard guard(ctx->device);
  a.num_orders = B;
  a.orders = d_orders;
  a.edge_src = g->d_edge_src;
  a.sink_off = g->d_sink_off;
  a.sinks = g->d_sinks;
  a.edge_size = g->d_edge_size;
  a.edge_size32 = std::getenv("MP_ARENA_WIDE_SIZE") ? nullptr : g->d_edge_size32;
  a.scale = a.edge_size32 ? g->scale : 1;  // 64-bit block sizes are bytes
  a.out_off = g->d_out_off;
  a.out_edges = g->d_out_edges;
  a.best_fit = best_fit ? 1 : 0;
  a.mr_peak = d_mr;
  a.rs_at_peak = d_rs;
  a.frag = d_frag;
  a.valid = d_valid;
  return launch_arena(a, ctx, static_cast<cudaStream_t>(stream));
}

mp_status mp_run_baseline(mp_ctx* ctx, const mp_graph* g, const int32_t* orders, int64_t B,
                          int best_fit, uint64_t* mr, uint64_t* rs, double* frag,
                          uint8_t* valid) {
  MP_TRY(same_ctx(ctx, g));
  if (!ctx || !g || B < 0) return invalid_arg("null argument");
  if (B == 0) return MP_OK;
  if ((!orders && g->n > 0) || !mr || !rs || !frag || !valid) return invalid_arg("null argument");
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t b = (size_t)B, on = b * (size_t)g->n;
  MP_TRY(ctx->scratch[0].reserve(Carver::size_of({4 * on, 8 * b, 8 * b, 8 * b, b})));
  Carver cv(ctx->scratch[0].ptr);
  int32_t* d_o = cv.take<int32_t>(on);
  uint64_t* d_mr = cv.take<uint64_t>(b);
  uint64_t* d_rs = cv.take<uint64_t>(b);
  double* d_fr = cv.take<double>(b);
  uint8_t* d_v = cv.take<uint8_t>(b);
  if (on) MP_CUDA(cudaMemcpyAsync(d_o, orders, 4 * on, cudaMemcpyHostToDevice, st));
  MP_TRY(mp_run_baseline_d(ctx, g, d_o, B, best_fit, d_mr, d_rs, d_fr, d_v, st));
  MP_CUDA(cudaMemcpyAsync(mr, d_mr, 8 * b, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaMemcpyAsync(rs, d_rs, 8 * b, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaMemcpyAsync(frag, d_fr, 8 * b, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaMemcpyAsync(valid, d_v, b, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  return MP_OK;
}

// ---- placement (K5) ---------------------------------------------------------------
static mp_status place_check(int32_t E, int64_t B, uint32_t flags, const void* fixed) {
  if (E < 0 || B < 0) return invalid_arg("negative size");
  if ((flags & (MP_PLACE_PYRAMID | MP_PLACE_PYRAMID_ONLY)) && fixed)
    return invalid_arg("a preplaced map and MP_PLACE_PYRAMID are exclusive");
  if (E > kPlaceBigMaxEdges) {
    set_error("Capacity: " + std::to_string(E) + " edges exceed the placement kernels' " +
              std::to_string(kPlaceBigMaxEdges) + " per problem");
    return MP_E_CAPACITY;
  }
  return MP_OK;
}

mp_status mp_place_d(mp_ctx* ctx, int32_t E, int64_t B, const int32_t* d_lo, const int32_t* d_hi,
                     const uint64_t* d_size, const int32_t* d_id_rank, const uint8_t* d_fixed,
                     const uint64_t* d_fixed_addr, uint32_t flags, uint64_t* d_addr,
                     uint8_t* d_has_addr, uint64_t* d_peak_mem, uint64_t* d_pyramid_base,
                     void* stream) {
  if (!ctx) return invalid_arg("null context");
  MP_TRY(place_check(E, B, flags, d_fixed));
  if (E > 0 && B > 0 && (!d_lo || !d_hi || !d_size || !d_addr || !d_has_addr))
    return invalid_arg("null argument");
  if (d_fixed && !d_fixed_addr) return invalid_arg("fixed without fixed_addr");
  DeviceGuard guard(ctx->device);
  PlaceArgs a;
  a.num_edges = E;
  a.num_problems = B;
  a.lo = d_lo;
  a.hi = d_hi;
  a.size = d_size;
  a.id_rank = d_id_rank;
  a.fixed = d_fixed;
  a.fixed_addr = d_fixed_addr;
  a.pyramid = (flags & (MP_PLACE_PYRAMID | MP_PLACE_PYRAMID_ONLY)) ? 1 : 0;
  a.pyramid_only = (flags & MP_PLACE_PYRAMID_ONLY) ? 1 : 0;
  a.addr = d_addr;
  a.has_addr = d_has_addr;
  a.peak_mem = d_peak_mem;
  a.pyramid_base = d_pyramid_base;
  return launch_place(a, ctx, static_cast<cudaStream_t>(stream));
}

mp_status mp_lifetimes_batch_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_orders,
                               int64_t C, int32_t* d_lo, int32_t* d_hi, uint8_t* d_valid,
                               void* stream) {
  if (!ctx || !g || C < 0) return invalid_arg("null argument or negative count");
  if (g->ctx != ctx) return invalid_arg("graph belongs to another context");
  if (C > 0 && ((g->n > 0 && !d_orders) || !d_valid || (g->E > 0 && (!d_lo || !d_hi))))
    return invalid_arg("null buffer");
  DeviceGuard guard(ctx->device);
  const mp_status s = launch_lifetimes_batch(g, d_orders, C, d_lo, d_hi, d_valid,
                                             static_cast<cudaStream_t>(stream));
  if (s == MP_E_CAPACITY) set_error("Capacity: graph too large for the batched lifetimes kernel");
  return s;
}

mp_status mp_validate_plans_d(mp_ctx* ctx, int32_t E, int64_t C, const int32_t* d_lo,
                              const int32_t* d_hi, const uint64_t* d_size, const uint8_t* d_has,
                              const uint64_t* d_addr, const uint8_t* d_valid, uint32_t* d_nviol,
                              void* stream) {
  if (!ctx || E < 0 || C < 0) return invalid_arg("null argument or negative count");
  if (C > 0 && (!d_nviol || (E > 0 && (!d_lo || !d_hi || !d_size || !d_has || !d_addr))))
    return invalid_arg("null buffer");
  if (E > kPlaceMaxEntries) {
    set_error("Capacity: the batched address check handles at most 8192 edges per plan");
    return MP_E_CAPACITY;
  }
  DeviceGuard guard(ctx->device);
  return launch_plan_check(ctx, C, E, d_lo, d_hi, d_size, d_has, d_addr, d_valid, d_nviol, nullptr,
                           static_cast<cudaStream_t>(stream));
}

mp_status mp_score_plans_d(mp_ctx* ctx, const mp_graph* g, const int32_t* d_orders, int64_t C,
                           const int32_t* d_id_rank, uint32_t flags, uint64_t* d_peak_rs,
                           int32_t* d_peak_step, uint8_t* d_valid, uint64_t* d_peak_mem,
                           uint32_t* d_nviol, uint64_t* d_addr, uint8_t* d_has,
                           uint64_t* d_best_key, int64_t index_base, void* stream) {
  if (!ctx || !g || C < 0 || index_base < 0) return invalid_arg("null argument or negative count");
  if (g->ctx != ctx) return invalid_arg("graph belongs to another context");
  if (flags & ~MP_PLACE_PYRAMID) return invalid_arg("flags: only MP_PLACE_PYRAMID is accepted");
  if (C > 0 && (!d_peak_rs || !d_peak_step || !d_valid || !d_peak_mem || !d_nviol ||
                (g->n > 0 && !d_orders)))
    return invalid_arg("null buffer");
  if (g->E > kPlaceBigMaxEdges) {
    set_error("Capacity: placement handles at most " + std::to_string(kPlaceBigMaxEdges) +
              " edges per problem");
    return MP_E_CAPACITY;
  }
  if (C == 0) return MP_OK;
  DeviceGuard guard(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t E = (size_t)g->E, c = (size_t)C, n = (size_t)g->n;
  // graphs past the shared-memory kernels (lifetimes, placed set, pair records): K1 per
  // candidate, K5's global-memory variant, the K4 sweep per plan
  const bool large = g->E > kPlaceMaxEntries || lifetimes_batch_smem(g->n) > ctx->max_smem_optin ||
                     plan_check_smem(g->E) > ctx->max_smem_optin;
  MP_TRY(ctx->scratch[6].reserve(Carver::size_of(
      {4 * E * c, 4 * E * c, c, d_addr ? 0 : 8 * E * c, d_has ? 0 : E * c, large ? 4 * c : 0,
       large ? 4 * (n + 1) : 0, large ? 8 * (E + 1) : 0})));
  Carver cv(ctx->scratch[6].ptr);
  int32_t* d_lo = cv.take<int32_t>(E * c);
  int32_t* d_hi = cv.take<int32_t>(E * c);
  uint8_t* d_lv = cv.take<uint8_t>(c);
  if (!d_addr) d_addr = cv.take<uint64_t>(E * c);
  if (!d_has) d_has = cv.take<uint8_t>(E * c);
  // the schedules (K3), their lifetimes, their placements, the address check, the key
  MP_TRY(launch_score(g, d_orders, C, d_peak_rs, d_peak_step, d_valid, nullptr, nullptr, 0, st));
  if (large) {
    int32_t* d_lv32 = cv.take<int32_t>(c);
    int32_t* d_pos = cv.take<int32_t>(n + 1);
    int64_t* d_row_off = cv.take<int64_t>(E + 1);
    MP_TRY(launch_lifetimes_large(g, d_orders, C, d_lo, d_hi, d_lv32, d_lv, d_pos, st));
    PlaceArgs a;
    a.num_edges = g->E;
    a.num_problems = C;
    a.lo = d_lo;
    a.hi = d_hi;
    a.size = g->d_edge_size;
    a.id_rank = d_id_rank;
    a.pyramid = (flags & MP_PLACE_PYRAMID) ? 1 : 0;
    a.addr = d_addr;
    a.has_addr = d_has;
    a.peak_mem = d_peak_mem;
    MP_TRY(launch_place(a, ctx, st));
    MP_TRY(launch_plan_check_large(ctx, C, g->E, d_lo, d_hi, g->d_edge_size, d_has, d_addr, d_lv,
                                   d_nviol, d_peak_mem, d_row_off, st));
    if (d_best_key)
      MP_TRY(launch_plan_key(C, d_lv, d_nviol, d_peak_mem, index_base, d_best_key, st));
    return MP_OK;
  }
  mp_status s = launch_lifetimes_batch(g, d_orders, C, d_lo, d_hi, d_lv, st);
  if (s == MP_E_CAPACITY) set_error("Capacity: graph too large for the batched lifetimes kernel");
  MP_TRY(s);
  PlaceArgs a;
  a.num_edges = g->E;
  a.num_problems = C;
  a.lo = d_lo;
  a.hi = d_hi;
  a.size = g->d_edge_size;
  a.id_rank = d_id_rank;
  a.pyramid = (flags & MP_PLACE_PYRAMID) ? 1 : 0;
  a.addr = d_addr;
  a.has_addr = d_has;
  a.peak_mem = d_peak_mem;
  MP_TRY(launch_place(a, ctx, st));
  MP_TRY(launch_plan_check(ctx, C, g->E, d_lo, d_hi, g->d_edge_size, d_has, d_addr, d_lv, d_nviol,
                           d_peak_mem, st));
  if (d_best_key) MP_TRY(launch_plan_key(C, d_lv, d_nviol, d_peak_mem, index_base, d_best_key, st));
  return MP_OK;
}

mp_status mp_place(mp_ctx* ctx, int32_t E, int64_t B, const int32_t* lo, const int32_t* hi,
                   const uint64_t* size, const int32_t* id_rank, const uint8_t* fixed,
                   const uint64_t* fixed_addr, uint32_t flags, uint64_t* addr, uint8_t* has_addr,
                   uint64_t* peak_mem, uint64_t* pyramid_base) {
  if (!ctx) return invalid_arg("null context");
  MP_TRY(place_check(E, B, flags, fixed));
  if (E == 0 || B == 0) {
    for (int64_t b = 0; b < B; ++b) {
      if (peak_mem) peak_mem[b] = 0;
      if (pyramid_base) pyramid_base[b] = 0;
    }
    return MP_OK;
  }
  if (!lo || !hi || !size || !addr || !has_addr) return invalid_arg("null argument");
  if (fixed && !fixed_addr) return invalid_arg("fixed without fixed_addr");
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t e = (size_t)E, be = (size_t)B * e, b = (size_t)B;
  MP_TRY(ctx->scratch[0].reserve(
      Carver::size_of({4 * be, 4 * be, 8 * e, 4 * e, e, 8 * e, 8 * be, be, 8 * b, 8 * b})));
  Carver cv(ctx->scratch[0].ptr);
  int32_t* d_lo = cv.take<int32_t>(be);
  int32_t* d_hi = cv.take<int32_t>(be);
  uint64_t* d_size = cv.take<uint64_t>(e);
  int32_t* d_rank = cv.take<int32_t>(e);
  uint8_t* d_fixed = cv.take<uint8_t>(e);
  uint64_t* d_faddr = cv.take<uint64_t>(e);
  uint64_t* d_addr = cv.take<uint64_t>(be);
  uint8_t* d_has = cv.take<uint8_t>(be);
  uint64_t* d_peak = cv.take<uint64_t>(b);
  uint64_t* d_base = cv.take<uint64_t>(b);
  MP_CUDA(cudaMemcpyAsync(d_lo, lo, 4 * be, cudaMemcpyHostToDevice, st));
  MP_CUDA(cudaMemcpyAsync(d_hi, hi, 4 * be, cudaMemcpyHostToDevice, st));
  MP_CUDA(cudaMemcpyAsync(d_size, size, 8 * e, cudaMemcpyHostToDevice, st));
  if (id_rank) MP_CUDA(cudaMemcpyAsync(d_rank, id_rank, 4 * e, cudaMemcpyHostToDevice, st));
  if (fixed) {
    MP_CUDA(cudaMemcpyAsync(d_fixed, fixed, e, cudaMemcpyHostToDevice, st));
    MP_CUDA(cudaMemcpyAsync(d_faddr, fixed_addr, 8 * e, cudaMemcpyHostToDevice, st));
  }
  MP_TRY(mp_place_d(ctx, E, B, d_lo, d_hi, d_size, id_rank ? d_rank : nullptr,
                    fixed ? d_fixed : nullptr, fixed ? d_faddr : nullptr, flags, d_addr, d_has,
                    d_peak, d_base, st));
  MP_TRY(d2h_large(ctx, addr, d_addr, 8 * be, st));  // the address plans: B x E x 8 bytes
  MP_CUDA(cudaMemcpyAsync(has_addr, d_has, be, cudaMemcpyDeviceToHost, st));
  if (peak_mem) MP_CUDA(cudaMemcpyAsync(peak_mem, d_peak, 8 * b, cudaMemcpyDeviceToHost, st));
  if (pyramid_base)
    MP_CUDA(cudaMemcpyAsync(pyramid_base, d_base, 8 * b, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  return MP_OK;
}

mp_status mp_addresses_feasible(mp_ctx* ctx, int32_t E, const int32_t* lo, const int32_t* hi,
                                const uint64_t* size, const uint8_t* has_addr,
                                const uint64_t* addr, int32_t* feasible) {
  if (!feasible) return invalid_arg("feasible is null");
  int64_t cnt = 0;
  MP_TRY(pair_sweep_h(ctx, 1, E, lo, hi, size, has_addr, addr, nullptr, 0, &cnt));
  *feasible = cnt == 0 ? 1 : 0;
  return MP_OK;
}

mp_status mp_peak_mem(mp_ctx* ctx, int32_t E, const uint64_t* size, const uint8_t* has_addr,
                      const uint64_t* addr, uint64_t* peak_mem) {
  if (!ctx || !peak_mem || E < 0 || (E > 0 && (!size || !has_addr || !addr)))
    return invalid_arg("null argument");
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t e = (size_t)E;
  MP_TRY(ctx->scratch[0].reserve(Carver::size_of({8 * e, e, 8 * e, 8})));
  Carver cv(ctx->scratch[0].ptr);
  uint64_t* d_size = cv.take<uint64_t>(e);
  uint8_t* d_has = cv.take<uint8_t>(e);
  uint64_t* d_addr = cv.take<uint64_t>(e);
  uint64_t* d_out = cv.take<uint64_t>(1);
  if (e) {
    MP_CUDA(cudaMemcpyAsync(d_size, size, 8 * e, cudaMemcpyHostToDevice, st));
    MP_CUDA(cudaMemcpyAsync(d_has, has_addr, e, cudaMemcpyHostToDevice, st));
    MP_CUDA(cudaMemcpyAsync(d_addr, addr, 8 * e, cudaMemcpyHostToDevice, st));
  }
  MP_TRY(launch_peak_mem(E, d_size, d_has, d_addr, d_out, st));
  MP_CUDA(cudaMemcpyAsync(peak_mem, d_out, 8, cudaMemcpyDeviceToHost, st));
  MP_CUDA(cudaStreamSynchronize(st));
  return MP_OK;
}

double mp_fragmentation(uint64_t mr, uint64_t rs) {
  // placement.cpp:64-67, the same expression on the host (one FP divide).
  if (mr == 0) return 0.0;
  return static_cast<double>(mr - rs) / static_cast<double>(mr);
}

}  // extern "C"
