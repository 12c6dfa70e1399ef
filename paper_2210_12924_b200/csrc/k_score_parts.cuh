// Node-partitioned large-graph scorer (MP_SCORER_PARTS), included by
// k_score.cu inside namespace mpb::{anon}. Host planning: mp_parts.cpp.
//
// One 1024-thread CTA per SM scores one candidate at a time (persistent). The
// candidate's positions never leave the SM: in pass b (one per node part) the
// CTA streams the order row (coalesced int4 loads; pass 0 from HBM, the rest
// from L2) and keeps only part b's nodes. One 32-bit shared word per local slot
// holds the node's static scan input ((x + 8) | f << 4, set at the start of the
// pass) in its low byte and its 1-based position in the top 24 bits
// (0xffffff = not written this pass):
//     w = slot[local(v)]; slot[local(v)] = (k + 1) << 8 | (w & 0xff);  XF[k] = (uint8_t)w
// Position on top lets every lookup compare or max whole words: two written slots
// differ in position, and an unwritten one fails the permutation check anyway.
// Then every lookup of part b resolves in shared memory: the permutation check
// (each local slot written this pass), the validity pairs inside the part, the
// cross-part pairs through a stash slot written by the earlier part, and the
// multi-consumer tensors (hi = max over the candidate sinks -> the free lands on
// XF[hi] with one global atomic). After the last pass a blocked scan over XF
// (global, L2-resident, 1 B per position) gives RS(p), the peak and the first
// step attaining it, as the other variants (schedule.cpp:69-88, plan.cpp:135-141).
//
// Per candidate the only global traffic is the order (4n B from HBM once, then
// from L2 per extra pass), XF (n B written, n B read), one atomic per
// multi-consumer tensor and the static lists (shared by all CTAs, L2-resident).
// The scratch variant instead spends a 32-byte L2 sector on each of ~3.5
// random 4-byte position accesses per node.

struct PartArgs {
  int32_t P, nchunks, nb_max, nslots, seg;
  int32_t n_slot_init, n_xfree;
  const PartDesc* __restrict__ desc;
  const uint32_t* __restrict__ ctab;
  const uint8_t* __restrict__ xtab;
  const uint16_t* __restrict__ p1;
  const uint32_t* __restrict__ intra;
  const uint32_t* __restrict__ xput;
  const uint32_t* __restrict__ xchk;
  const uint32_t* __restrict__ xmax;
  const uint4* __restrict__ dyn4;
  const uint2* __restrict__ xfree;
  const int32_t* __restrict__ slot_init;
};

constexpr int kPartsThreads = 1024;
#ifndef MP_PARTS_U
#define MP_PARTS_U 4
#endif
constexpr int kPartsU = MP_PARTS_U;  // 16-byte order loads per thread per stream iteration
constexpr int kPartsMaxBlocks = 512;  // kDefer: 512-position blocks (n <= 262,144)
#ifndef MP_SCAN_U
#define MP_SCAN_U 3
#endif
constexpr int kScanU = MP_SCAN_U;  // 16-byte XF loads in flight per lane in the scan
#ifndef MP_LOOK_U
#define MP_LOOK_U 4
#endif
constexpr int kLookU = MP_LOOK_U;  // first-producer / two-sink groups' loads in flight

__device__ __forceinline__ size_t parts_al16(size_t b) { return (b + 15) & ~size_t(15); }

// The free of a multi-consumer tensor after position hi: x -= sz, f += sz on the
// 4-bit pair, i.e. +15*sz on the byte (no carry leaves it: tiny4 bounds every
// order); on the 32-bit word that holds it, at L2.
__device__ __forceinline__ void parts_free_at(uint8_t* XF, int hi, uint32_t sz) {
  atomicAdd(reinterpret_cast<unsigned int*>(XF + (hi & ~3)), (sz * 15u) << ((hi & 3) * 8));
}

__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
  asm volatile("" : "+r"(v));
  return v;
}
__device__ __forceinline__ uint64_t opaque_u64(uint64_t v) {
  asm volatile("" : "+l"(v));
  return v;
}
__device__ __forceinline__ void stg_u8(uint8_t* p, uint32_t v) {
  asm volatile("st.global.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// 32-bit shared-window accesses (addresses computed once, not per generic access)
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// k24: orders arrive as 24-bit ids (3 bytes per position, host-packed for the
// PCIe leg of the host-buffer call; n % 4 == 0, out-of-range ids as 0xffffff).
// kDefer: the order is streamed ONCE, in 512-position blocks that the warps take
// from a shared counter. Pass 0 keeps part 0's positions and appends every other
// in-range position to its block's deferred list in global scratch (L2-resident),
// one word {local slot, position - block start, part}; pass b >= 1 takes the blocks'
// lists the same way instead of the order and the chunk table, and keeps part b's
// words (needs P <= 7 - part 7 marks nothing - and n <= 512 * kPartsMaxBlocks).
// Measured: one list read by every later pass beats one list per part (two ballots
// per position to append) at C5.
// MP_PARTS_PROF (a profiling build only): thread 0 of CTA 0 accumulates the clock cycles
// between the phase barriers and prints them at exit
#ifdef MP_PARTS_PROF
#define MP_PARTS_T0() \
  unsigned long long prof_acc[15] = {}, prof_last = clock64();
#define MP_PARTS_T(i)                                  \
  if (tid == 0) {                                      \
    const unsigned long long t_ = clock64();           \
    prof_acc[(i)] += t_ - prof_last;                   \
    prof_last = t_;                                    \
  }
#else
#define MP_PARTS_T0()
#define MP_PARTS_T(i)
#endif

template <bool kVec, bool k24 = false, bool kDefer = false>
__global__ void __launch_bounds__(kPartsThreads, 1)
    score_parts_kernel(PartArgs A, int32_t n, const int32_t* __restrict__ orders, int64_t C,
                       uint64_t* __restrict__ peak_out, int32_t* __restrict__ step_out,
                       uint8_t* __restrict__ valid_out, unsigned long long* __restrict__ best_key,
                       int64_t index_base, uint64_t scale, uint8_t* __restrict__ gxf,
                       size_t gstride, size_t xf_bytes) {
  extern __shared__ __align__(16) char smem[];
  __shared__ uint32_t s_wsum[32];
  __shared__ uint32_t s_bcnt[kPartsMaxBlocks];  // kDefer: deferred words per 512-position block
  __shared__ uint32_t s_next[kPartMaxParts];    // kDefer: next block to take, per pass
  __shared__ uint32_t s_wbest[32];
  __shared__ int s_widx[32];
  __shared__ PartDesc s_desc[kPartMaxParts];  // read field by field where used (registers)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int T = kPartsThreads;
  constexpr uint32_t kPos = 0xffffffu;  // chunk-table local base bits
  constexpr uint32_t kUnw = 0xffffff00u;  // slot words >= this: not written this pass
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem);
  uint32_t* ctab_s = reinterpret_cast<uint32_t*>(smem + parts_al16((size_t)(A.nb_max + 2) * 4));
  uint32_t* stash = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(ctab_s) +
                                                parts_al16((size_t)(A.nchunks + 1) * 4));
  // kept in registers (opaque to the compiler, which would otherwise rematerialise
  // the shared window base and the scratch pointer inside every member branch)
  const uint32_t slot_a = opaque_u32((uint32_t)__cvta_generic_to_shared(slot));
  const uint32_t ctab_a = opaque_u32((uint32_t)__cvta_generic_to_shared(ctab_s));
  uint8_t* XF = reinterpret_cast<uint8_t*>(
      opaque_u64(reinterpret_cast<uint64_t>(gxf + (size_t)blockIdx.x * gstride)));
  const int seg = A.seg;  // positions per warp segment, a multiple of 512 (lane chunks of 16-byte multiples)
  const int wbeg = warp * seg;
  const int wend = wbeg + seg;   // loops run in 512-position steps and stop at wend
  const int wlim = min(n, wend);  // this warp's real positions end here
  // kDefer: block t's deferred words (at most 512) at dbase + 512 t
  uint32_t* dbase = reinterpret_cast<uint32_t*>(
      opaque_u64(reinterpret_cast<uint64_t>(gxf + (size_t)blockIdx.x * gstride + xf_bytes)));
  const uint32_t nblk = (uint32_t)(n + 511) >> 9;

  // kDefer keeps the chunk table pre-formatted as a deferred word: part << 29 | local base
  // (parts past P - out-of-range ids - become part 7, which no pass keeps)
  for (int i = tid; i <= A.nchunks; i += T) {
    const uint32_t e = __ldg(A.ctab + i);
    ctab_s[i] = !kDefer ? e : ((e >> 24) < (uint32_t)A.P ? (e >> 24) : 7u) << 29 | (e & 0xffffffu);
  }
  if (tid < A.P) s_desc[tid] = A.desc[tid];
  for (int i = n + tid; i < 32 * seg; i += T) XF[i] = 8;  // scan padding: x = 0, f = 0
  // sentinel slots (positions are 1-based): nb_max reads position 0 ("no producer",
  // "no sink"), nb_max + 1 reads unwritten (the padding pair of the intra lists)
  if (tid == 0) {
    slot[A.nb_max] = 0;
    slot[A.nb_max + 1] = kUnw;
  }
  __syncthreads();
  MP_PARTS_T0();

  for (int64_t c = blockIdx.x; c < C; c += gridDim.x) {
    const int32_t* ord = orders + c * (int64_t)n;
    // 24-bit rows: 3n bytes each = 3n/4 words (n % 4 == 0)
    const uint32_t* ord24 = reinterpret_cast<const uint32_t*>(orders) + c * (int64_t)(3 * (n >> 2));
    bool bad = false;
    if (kDefer && tid < kPartMaxParts) s_next[tid] = 0;  // read after pass 0's slot init barrier
    for (int i = tid; i < A.n_slot_init; i += T) stash[__ldg(A.slot_init + i)] = 0;

    for (int b = 0; b < A.P; ++b) {
      const PartDesc& D = s_desc[b];
      {  // slot words: this part's static scan input on top, "not written" below
        // one xtab word -> four consecutive slot words per thread: 16-byte stores
        // of consecutive lanes are contiguous (no bank conflicts)
        const uint32_t* src = reinterpret_cast<const uint32_t*>(A.xtab + D.xtab_off);
        uint4* dst = reinterpret_cast<uint4*>(slot);
        // slots past the last node ([pad_lo, pad_hi), never written) start at position 1
        // (written, and after the position-0 sentinel of "no producer")
        // so the permutation check below needs no range test
        const int plo = D.pad_lo, phi = D.pad_hi;
        const int qlo = plo >> 2, qhi = (phi + 3) >> 2;  // uint4 words touching the pad
        const int nq = D.nloc >> 2;
        for (int i0 = tid; i0 < nq; i0 += 4 * T) {
          uint32_t ws[4];  // four words' loads in flight
#pragma unroll
          for (int u = 0; u < 4; ++u) ws[u] = i0 + u * T < nq ? __ldg(src + i0 + u * T) : 0u;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * T;
          if (i >= nq) break;
          const uint32_t w = ws[u];
          uint4 o = make_uint4(kUnw | (w & 0xffu), kUnw | ((w >> 8) & 0xffu),
                               kUnw | ((w >> 16) & 0xffu), kUnw | (w >> 24));
          if (i >= qlo && i < qhi) {
            const int l = 4 * i;
            if (l >= plo && l < phi) o.x = (o.x & 0xffu) | 0x100u;
            if (l + 1 >= plo && l + 1 < phi) o.y = (o.y & 0xffu) | 0x100u;
            if (l + 2 >= plo && l + 2 < phi) o.z = (o.z & 0xffu) | 0x100u;
            if (l + 3 >= plo && l + 3 < phi) o.w = (o.w & 0xffu) | 0x100u;
          }
          dst[i] = o;
          }
        }
      }
      __syncthreads();
      MP_PARTS_T(3 * min(b, 3));

      // ---- stream the order: keep part b's nodes -----------------------------------
      // 16 positions per thread per iteration: their chunk-table lookups are issued
      // together, then each member does one shared read-modify-write and one byte
      // store. A whole iteration of real positions only tracks the max id (range
      // check after the loop); the segment tail checks per position.
      const bool last = b == A.P - 1;
      const uint32_t bsel = (uint32_t)b << 24;
      if (kDefer && b > 0) {
        // the deferred words block by block, blocks taken from a shared counter (the
        // warps finish together); 4 words per 16-byte load, part b's kept
        for (;;) {
          uint32_t t = 0;
          if (lane == 0) t = atomicAdd(&s_next[b], 1u);
          t = __shfl_sync(0xffffffffu, t, 0);
          if (t >= nblk) break;
          const uint32_t cnt = s_bcnt[t];
          const uint32_t* dl = dbase + ((size_t)t << 9);
          const uint32_t kb = t << 9;
          const uint32_t nu = (cnt + 127u) >> 7;  // 128-word rows holding words (uniform)
          uint4 q[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            q[u] = 4 * lane + u * 128 < cnt
                       ? __ldcg(reinterpret_cast<const uint4*>(dl + 4 * lane + u * 128))
                       : make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if ((uint32_t)u >= nu) break;
            const uint32_t ev[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const uint32_t e = ev[h];
              if ((e >> 29) == (uint32_t)b) {  // groups past the end read as ~0
                const uint32_t a = slot_a + 4u * (e & 0xffffu);
                const uint32_t w = lds_u32(a);
                const uint32_t k = kb + ((e >> 16) & 0x1ffu);
                sts_u32(a, (k + 1) << 8 | (w & 0xffu));  // 1-based
                stg_u8(XF + k, w);
              }
            }
            // last reader: drop the consumed 128-byte lines from L2 without a write-back
            if (last && (lane & 7) == 0 && 4 * lane + u * 128 < cnt)
              asm volatile("discard.global.L2 [%0], 128;" ::"l"(dl + ((4 * lane + u * 128) & ~31u))
                           : "memory");
          }
        }
      } else
      for (int it = 0;; ++it) {
        // kDefer (pass 0): 512-position blocks from a shared counter (the warps finish
        // together); otherwise the warp's own segment in 512-position steps
        int r0, wlim_it;
        uint32_t t = 0;
        if (kDefer) {
          if (lane == 0) t = atomicAdd(&s_next[0], 1u);
          t = __shfl_sync(0xffffffffu, t, 0);
          if (t >= nblk) break;
          r0 = (int)(t << 9) + 4 * lane;
          wlim_it = n;
        } else {
          r0 = wbeg + 4 * lane + it * (kPartsU * 128);
          if (r0 >= wbeg + seg) break;
          wlim_it = wlim;
        }
        uint32_t vq[4 * kPartsU];
#pragma unroll
        for (int u = 0; u < kPartsU; ++u) {  // kPartsU 16-byte loads in flight per thread
          const int r = r0 + u * 128;
          int4 q;
          if (k24) {  // four 3-byte ids in three words (word index 3r/4)
            if (r >= wlim_it) {
              q = make_int4(-1, -1, -1, -1);
            } else {
              const uint32_t* w = ord24 + 3 * (r >> 2);
              const uint32_t w0 = __ldg(w), w1 = __ldg(w + 1), w2 = __ldg(w + 2);
              auto id = [](uint32_t x) { return x == 0xffffffu ? -1 : (int)x; };
              q = make_int4(id(w0 & 0xffffffu), id((w0 >> 24) | ((w1 & 0xffffu) << 8)),
                            id((w1 >> 16) | ((w2 & 0xffu) << 16)), id(w2 >> 8));
            }
          } else if (kVec) {
            const int4* p4 = reinterpret_cast<const int4*>(ord + r);
            q = r >= wlim_it ? make_int4(-1, -1, -1, -1) : (last || kDefer) ? __ldcs(p4) : __ldg(p4);
          } else {
            q.x = r < wlim_it ? __ldg(ord + r) : -1;
            q.y = r + 1 < wlim_it ? __ldg(ord + r + 1) : -1;
            q.z = r + 2 < wlim_it ? __ldg(ord + r + 2) : -1;
            q.w = r + 3 < wlim_it ? __ldg(ord + r + 3) : -1;
          }
          vq[4 * u] = (uint32_t)q.x, vq[4 * u + 1] = (uint32_t)q.y;
          vq[4 * u + 2] = (uint32_t)q.z, vq[4 * u + 3] = (uint32_t)q.w;
        }
        // no range check: an id outside [0, n) maps to the chunk table's "no part" entry,
        // so no pass writes it, and with n positions some node then stays unwritten - the
        // permutation check below rejects the order
        if (kDefer) {
          // pass 0: part 0 now, parts 1.. appended to the deferred list. One word per
          // position either way: {local, position - segment start, part}, ~0 out of range
          // the table word already is part << 29 | local base: add the id's offset in
          // its chunk and the position's offset in the segment (no carries: local
          // < 2^16, offset < 2^13)
          const uint32_t k16 = (uint32_t)(4 * lane) << 16;  // position - block start
#pragma unroll
          for (int j = 0; j < 4 * kPartsU; ++j) {
            const uint32_t e = lds_u32(ctab_a + 4u * min(vq[j] >> kPartChunkBits, (uint32_t)A.nchunks));
            vq[j] = e + (vq[j] & ((1u << kPartChunkBits) - 1)) +
                    (k16 + ((uint32_t)((j >> 2) * 128 + (j & 3)) << 16));
          }
          // appended in (j, lane) order with ballot ranks: each store instruction
          // writes one contiguous run of the list (coalesced)
          const uint32_t lt = (1u << lane) - 1u;
          const uint32_t nd = (uint32_t)(A.P - 1) << 29;  // parts 1 .. P-1
          uint32_t bc = 0;                                // this block's deferred words
#pragma unroll
          for (int j = 0; j < 4 * kPartsU; ++j) {
            const uint32_t w = vq[j];
            const bool d = w - (1u << 29) < nd;
            const uint32_t bal = __ballot_sync(0xffffffffu, d);
            if (d) __stcg(dbase + ((size_t)t << 9) + bc + __popc(bal & lt), w);
            bc += __popc(bal);
            vq[j] = w < (1u << 29) ? w & 0xffffu : 0xffffffffu;  // part 0: this pass
          }
          // padded to whole 16-byte groups with ~0 (part 7: no pass keeps it), so the
          // readers test only the group, not every word, against the count
          if (lane < ((4u - (bc & 3u)) & 3u)) __stcg(dbase + ((size_t)t << 9) + bc + lane, ~0u);
          if (lane == 0) s_bcnt[t] = bc;
        } else {
          // id -> local slot of part b, or ~0 (another part / out of range), in place
#pragma unroll
          for (int j = 0; j < 4 * kPartsU; ++j) {
            const uint32_t e = lds_u32(ctab_a + 4u * min(vq[j] >> kPartChunkBits, (uint32_t)A.nchunks));
            vq[j] = (e ^ bsel) < (1u << 24) ? (e & kPos) + (vq[j] & ((1u << kPartChunkBits) - 1))
                                            : 0xffffffffu;
          }
        }
        uint8_t* xrow = XF + r0;
#pragma unroll
        for (int j = 0; j < 4 * kPartsU; ++j) {
          if (vq[j] != 0xffffffffu) {  // part b owns this position's node
            const uint32_t a = slot_a + 4u * vq[j];
            const uint32_t w = lds_u32(a);
            sts_u32(a, (uint32_t)(r0 + (j >> 2) * 128 + (j & 3) + 1) << 8 | (w & 0xffu));  // 1-based
            stg_u8(xrow + (j >> 2) * 128 + (j & 3), w);
          }
        }
      }
      __syncthreads();
      MP_PARTS_T(3 * min(b, 3) + 1);

      // ---- resolve part b's lookups in shared memory ---------------------------------
      // (a slot left unwritten stays >= kUnw: it fails the permutation check, so the
      // comparisons below never need to tell it apart)
      {  // every local node written this pass (a permutation), and its same-part
         // first producer strictly earlier: own words in 16-byte reads, producer ids
         // 4 x 16 bits per 8-byte load, one random slot read per node
        const uint4* sw = reinterpret_cast<const uint4*>(slot);
        const uint2* p1 = reinterpret_cast<const uint2*>(A.p1 + D.xtab_off);
        const int nq = D.nloc >> 2;
        for (int i0 = tid; i0 < nq; i0 += kLookU * T) {  // kLookU groups' loads in flight
          uint2 pp[kLookU];
#pragma unroll
          for (int u = 0; u < kLookU; ++u)
            pp[u] = i0 + u * T < nq ? __ldg(p1 + i0 + u * T) : make_uint2(~0u, ~0u);
#pragma unroll
          for (int u = 0; u < kLookU; ++u) {
            const int i = i0 + u * T;
            if (i >= nq) break;
            const uint4 q = sw[i];
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
            const uint32_t pr[4] = {pp[u].x & 0xffffu, pp[u].x >> 16, pp[u].y & 0xffffu,
                                    pp[u].y >> 16};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              bad |= w[h] >= kUnw;
              bad |= slot[pr[h]] >= w[h];  // none: the position-0 sentinel (word 0)
            }
          }
        }
      }
      // the static lists come as uint4 groups, two groups in flight per thread
      auto groups = [&](const uint32_t* list, int off, int cnt, auto&& fn) {
        const uint4* g4 = reinterpret_cast<const uint4*>(list) + off;
        for (int i = tid; i < cnt; i += 2 * T) {
          const uint4 g0 = __ldg(g4 + i);
          const uint4 g1 = i + T < cnt ? __ldg(g4 + i + T) : make_uint4(~0u, ~0u, ~0u, ~0u);
          const uint32_t es[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
          for (int h = 0; h < 8; ++h)
            if (es[h] != 0xffffffffu) fn(es[h]);
        }
      };
      {  // same-part validity pairs beyond p1, padded with the sentinel pair (no test)
        const uint4* g4 = reinterpret_cast<const uint4*>(A.intra) + D.intra_off;
        const uint32_t sp = (uint32_t)A.nb_max | (uint32_t)(A.nb_max + 1) << 16;
        for (int i = tid; i < D.intra_n; i += 2 * T) {
          const uint4 g0 = __ldg(g4 + i);
          const uint4 g1 = i + T < D.intra_n ? __ldg(g4 + i + T) : make_uint4(sp, sp, sp, sp);
          const uint32_t es[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
          for (int h = 0; h < 8; ++h)  // producer later
            bad |= slot[es[h] & 0xffffu] >= slot[es[h] >> 16];
        }
      }
      groups(A.xput, D.xput_off, D.xput_n,
             [&](uint32_t e) { stash[e >> 16] = slot[e & 0xffffu] >> 8; });
      groups(A.xchk, D.xchk_off, D.xchk_n, [&](uint32_t e) {
        const uint32_t s = stash[(e >> 16) & 0x7fffu];
        const uint32_t p = slot[e & 0xffffu] >> 8;
        if ((e >> 31) ? p >= s : s >= p) bad = true;
      });
      groups(A.xmax, D.xmax_off, D.xmax_n,
             [&](uint32_t e) { atomicMax(&stash[e >> 16], slot[e & 0xffffu] >> 8); });
      for (int i = tid; i < D.dyn_n; i += 4 * T) {  // multi-consumer tensors inside the part
        uint4 dd[4];  // four records' loads in flight
#pragma unroll
        for (int u = 0; u < 4; ++u)
          dd[u] = i + u * T < D.dyn_n ? __ldg(A.dyn4 + D.dyn_off + i + u * T) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint4 d = dd[u];
          if (d.z == 0) continue;  // padding (every real record frees >= 1 unit)
          const uint32_t l1 = d.x & 0xffffu, l2 = d.x >> 16, l3 = d.y & 0xffffu, l4 = d.y >> 16;
          // missing sinks read the position-0 sentinel
          const uint32_t h = max(max(slot[l1], slot[l2]), max(slot[l3], slot[l4])) >> 8;
          const uint32_t hi = h - 1u;  // 1-based; unwritten (invalid orders) or 0 -> skipped
          if (hi < (uint32_t)n) parts_free_at(XF, (int)hi, d.z);
        }
      }
      const uint32_t s2 = (uint32_t)A.nb_max * 0x10001u;  // both sinks: position 0
      for (int i = tid; i < D.dyn2_n; i += kLookU * T) {  // two-sink tensors, two per 16 bytes
        uint4 dd[kLookU];
#pragma unroll
        for (int u = 0; u < kLookU; ++u)  // past the end: the sentinel pair (no free)
          dd[u] = i + u * T < D.dyn2_n ? __ldg(A.dyn4 + D.dyn2_off + i + u * T)
                                       : make_uint4(s2, 0, s2, 0);
#pragma unroll
        for (int u = 0; u < kLookU; ++u) {
          const uint32_t ha = (max(slot[dd[u].x & 0xffffu], slot[dd[u].x >> 16]) >> 8) - 1u;
          const uint32_t hb = (max(slot[dd[u].z & 0xffffu], slot[dd[u].z >> 16]) >> 8) - 1u;
          if (ha < (uint32_t)n) parts_free_at(XF, (int)ha, dd[u].y);
          if (hb < (uint32_t)n) parts_free_at(XF, (int)hb, dd[u].w);
        }
      }
      __syncthreads();  // slot words are rewritten by the next pass
      MP_PARTS_T(3 * min(b, 3) + 2);
    }
    for (int i = tid; i < A.n_xfree; i += T) {  // multi-consumer tensors spanning parts
      const uint2 f = __ldg(A.xfree + i);
      const uint32_t hi = stash[f.x] - 1u;  // 1-based positions
      if (hi < (uint32_t)n) parts_free_at(XF, (int)hi, f.y);
    }
    const bool any_bad = __syncthreads_or(bad);
    MP_PARTS_T(12);
    if (any_bad) {
      if (tid == 0) {
        peak_out[c] = 0;
        step_out[c] = 0;
        valid_out[c] = 0;
      }
      continue;
    }

    // ---- scan over XF (L2 only: the frees above were atomics at L2) -------------------
    // One pass: each warp scans its segment relative to the segment start (signed local
    // sums, |x| <= 8 per position), keeping its total and its first local maximum
    // (adding the segment's true starting RS moves every local value by the same
    // amount, so the arg-max is the same); warp 0 then adds the exclusive prefix of the
    // totals and takes the first maximum over the warps.
    // Lane chunks: lane L scans its own cs = seg / 32 consecutive positions of the warp's
    // segment sequentially (16-byte L2 loads, kScanU in flight), keeping its local total and
    // its first local maximum (strict >: a padding position, x = f = 0, never beats the
    // positions before it). One warp scan of the lane totals then shifts each lane's maximum
    // by the lane's exclusive prefix (the same shift for all of a lane's positions, so its
    // arg-max stands), and the warp arg-max (smallest index on ties) takes the first.
    // Against one warp scan per 128 positions this has no shuffle chain per row.
    const int cs = seg >> 5;  // a multiple of 16 (seg % 512 == 0)
    const int l0 = wbeg + lane * cs;
    int32_t run = 0;
    int32_t best = INT32_MIN;
    int best_i = l0;
    for (int r = 0; r < cs; r += 16 * kScanU) {
      uint4 q[kScanU];
#pragma unroll
      for (int u = 0; u < kScanU; ++u)  // past the chunk: padding (x 0, f 0)
        q[u] = r + 16 * u < cs ? __ldcg(reinterpret_cast<const uint4*>(XF + l0 + r + 16 * u))
                               : make_uint4(0x08080808u, 0x08080808u, 0x08080808u, 0x08080808u);
#pragma unroll
      for (int u = 0; u < kScanU; ++u) {
        const uint32_t ws[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
        for (int h = 0; h < 16; ++h) {
          const uint32_t byte = (ws[h >> 2] >> (8 * (h & 3))) & 0xffu;
          run += (int32_t)(byte & 0xfu) - 8;
          const int32_t rs = run + (int32_t)(byte >> 4);
          const bool better = rs > best;
          best = better ? rs : best;
          best_i = better ? l0 + r + 16 * u + h : best_i;
        }
      }
    }
    const int32_t incl = warp_incl_scan(run, lane);
    const int32_t carry = __shfl_sync(0xffffffffu, incl, 31);  // the segment's x total
    best += incl - run;  // RS relative to the segment start at the lane's maximum
    warp_argmax(best, best_i);
    // XF is rewritten by the next candidate: drop this segment's lines from L2 without
    // a write-back (not the line holding position n - its padding bytes persist)
    for (int l0 = wbeg + 128 * lane; l0 + 128 <= min(wend, n & ~127); l0 += 128 * 32)
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(XF + l0) : "memory");
    if (lane == 0) {
      s_wsum[warp] = (uint32_t)carry;  // the segment's x total
      s_wbest[warp] = (uint32_t)best;
      s_widx[warp] = best_i;
    }
    __syncthreads();
    MP_PARTS_T(13);
    if (warp == 0) {
      const uint32_t tot = s_wsum[lane];
      uint32_t v = warp_incl_scan(tot, lane) - tot + s_wbest[lane];  // RS at the local max
      int vi = s_widx[lane];
      warp_argmax(v, vi);
      if (lane == 0) {
        const uint64_t pk = (uint64_t)v * scale;
        peak_out[c] = pk;
        step_out[c] = vi + 1;
        valid_out[c] = 1;
        if (best_key) record_key(best_key, pk, (uint64_t)(c + index_base));
      }
    }
    // s_wsum / s_wbest are rewritten after >= 2 barriers of the next candidate
  }
#ifdef MP_PARTS_PROF
  if (tid == 0 && blockIdx.x == 0)
    for (int i = 0; i < 15; ++i) printf("MP_PARTS_PROF phase %d cycles %llu\n", i, prof_acc[i]);
#endif
}
