// ffx_slice.cu -- the snapshot / recovery kernel: fused copy + per-slice
// FNV-1a-64 (+ verify against a checksum table, + slot commit).
//
// Work unit: one warp task = 32*RPL consecutive slices of one region; lane l
// owns slices l, l+32, ... (FNV-1a is byte-serial, hash.cpp:102-110, so the
// parallelism is independent slice chains).  Each step moves KC x 128 bytes
// of every slice of the task:
//
//   full, aligned task (the bulk of any payload) -- tensor TMA: the region
//     is viewed as {128, nslices, slice_bytes/128} (3-D, KC > 1; the default
//     KC = 2) or {slice_bytes, nslices} (2-D, KC = 1) with row pitch
//     slice_bytes; one cp.async.bulk.tensor load brings a box of KC planes of
//     128 x (32*RPL) bytes (row j = slice j) into shared memory with 128-byte
//     swizzle (S stages, mbarrier complete_tx), one tensor store writes it to
//     the destination (local HBM, the NVLink peer's replica, or an NVSwitch
//     multicast range; twice for the dual-store double neighbour), and each
//     lane hashes its rows from shared memory, reading chunk w of row j at
//     (w ^ (j & 7)) so every LDS.128 phase is conflict-free.  No payload byte
//     passes through registers on the copy path.
//   ragged task (region tail, unaligned pointers) -- register path: 16-byte
//     loads / stores and a padded shared-memory transpose.
//
// Tasks are handed out last task first -- each warp's first task by its
// index, the rest dynamically (one atomic per task) -- so the latency-bound
// ragged tails overlap the bulk and the last wave does not idle SMs.
// Task-granular launches (one_shot) instead give every warp exactly one task
// and exit, so a low-priority batch yields SMs at every task boundary.
//
// Two configurations ship (launch_mode): the bulk one (32-slice tasks, one
// FNV chain per lane, 4 warps, 98 KB) for full-GPU launches, and an SM-lean
// one (64-slice tasks, two chains per lane, 8 warps, 130 KB) for CTA-capped
// scheduler batches inside a training step, which also stream their TMA
// traffic through L2 evict-first.  The round-1 tuning table and its env
// knobs exist only in FFX_DEV builds.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include <cudaTypedefs.h>

#include "ffx_device.cuh"
#include "ffx_kernels.h"

namespace ffx {

namespace {

// Tuning experiments (kernel variants, start-up stagger, claim order, store
// hints, cross-task prefetch, per-step proxy fences) are compiled only into
// development builds (make DEV=1 -> -DFFX_DEV); the product library carries
// one configuration per mode and none of their branches.
#ifdef FFX_DEV
constexpr bool kDev = true;
#else
constexpr bool kDev = false;
#endif

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Volatile so a row's loads issue back to back ahead of its hashing rather
// than being sunk next to their first use.
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

// 16 bytes at base+o, zero past `bytes`; byte loads when unaligned / ragged.
__device__ __forceinline__ uint4 load16(const uint8_t* base, uint64_t o, uint64_t bytes, bool al) {
  if (al && o + 16 <= bytes) return ld_stream(base + o);
  uint32_t w[4] = {0, 0, 0, 0};
  if (o < bytes) {
    const uint64_t n = umin64(bytes - o, 16);
    for (uint64_t b = 0; b < n; ++b) w[b >> 2] |= static_cast<uint32_t>(base[o + b]) << (8 * (b & 3));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ void store16(uint8_t* base, uint64_t o, uint64_t bytes, bool al,
                                        const uint4& v) {
  if (al && o + 16 <= bytes) {
    st_stream(base + o, v);
    return;
  }
  if (o < bytes) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    const uint64_t n = umin64(bytes - o, 16);
    for (uint64_t b = 0; b < n; ++b) base[o + b] = static_cast<uint8_t>(w[b >> 2] >> (8 * (b & 3)));
  }
}

// ---- TMA bulk copies + mbarriers (PTX) ------------------------------------------

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "FFX_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra FFX_WAIT;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
// 2-D tensor TMA (tile mode): one op moves a 128 x 32 box = 4 KB.
__device__ __forceinline__ void tensor_load(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tensor_store(const CUtensorMap* map, int x, int y, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(src)
               : "memory");
}
// 3-D variant: box {128, ROWS, KC} -- KC consecutive 128 B chunks of each
// slice per op, laid out in shared memory as KC planes of ROWS x 128 B.
__device__ __forceinline__ void tensor_load3(uint32_t dst, const CUtensorMap* map, int y, int z, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(y), "r"(z), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tensor_store3(const CUtensorMap* map, int y, int z, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(y), "r"(z), "r"(src)
               : "memory");
}
// Loads and stores with an L2 eviction-priority hint (evict_first): the
// snapshot streams its bytes through L2 exactly once, so inside a training
// step it should not displace the step's own working set (the GEMM operands).
__device__ __forceinline__ void tensor_load_h(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tensor_load3_h(uint32_t dst, const CUtensorMap* map, int y, int z, uint32_t bar,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(y), "r"(z), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tensor_store_h(const CUtensorMap* map, int x, int y, uint32_t src, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(src), "l"(pol)
               : "memory");
}
// The 3-D store with the hint (also the FFX_STORE_HINT experiment).
__device__ __forceinline__ void tensor_store3_hint(const CUtensorMap* map, int y, int z, uint32_t src,
                                                   uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(y), "r"(z), "r"(src), "l"(policy)
               : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---- slot commit ------------------------------------------------------------------

__device__ __forceinline__ void commit_begin(const SlotCommit& c) {
  if (threadIdx.x == 0) {
    SlotMeta* m = reinterpret_cast<SlotMeta*>(c.slot);
    const bool mc = c.mcast != 0;
    meta_st32(&m->magic, kSlotMagic, mc);
    meta_st64(&m->iteration, c.iteration, mc);
    meta_st64(&m->seq, c.seq, mc);
    meta_st32(&m->state, kSlotWriting, mc);
    __threadfence_system();
  }
  __syncthreads();
}

// Called by thread 0 after the whole CTA finished (and its bulk stores landed).
__device__ __forceinline__ void commit_end(const SlotCommit& c) {
  if (!c.finalize) return;
  __threadfence_system();
  const unsigned prev = atomicAdd(c.done, 1u);
  if (prev != gridDim.x - 1) return;
  __threadfence_system();
  const bool mc = c.mcast != 0;
  for (int i = 1; i < static_cast<int>(kMetaBytes / 16); ++i) meta_st128(c.slot + 16 * i, c.meta[i], mc);
  for (int i = 0; i < 2; ++i) meta_st128(c.slot + c.payload_off - 32 + 16 * i, c.snp1[i], mc);
  __threadfence_system();
  meta_st32(&reinterpret_cast<SlotMeta*>(c.slot)->state, kSlotCommitted, mc);
  __threadfence_system();
  if (c.ack != nullptr) {  // pull mode: release the origin's optimizer update
    *reinterpret_cast<volatile uint64_t*>(c.ack) = c.ack_value;
    __threadfence_system();
  }
  *c.done = 0;
}

template <int S, int W, int RPL, int KC>
struct Cfg {
  static constexpr int C = 128;                      // bytes of each slice per plane (one TMA row)
  static constexpr int VPL = C / 16;                 // 16-byte vectors per row
  static constexpr int ROWS = 32 * RPL;              // slices per warp task (RPL per lane)
  static constexpr int PLANE = ROWS * C;             // 128 x ROWS, dense + swizzled
  static constexpr int STAGE = PLANE * KC;           // one TMA box: KC planes
  static constexpr int PADROW = C + 16;              // register-path row, padded for banks
  static constexpr int WARPB = S * STAGE > 32 * PADROW ? S * STAGE : 32 * PADROW;
  // [tiles: W x WARPB, 1 KB-aligned (128 B swizzle atoms)][mbarriers: W x S x 8 B]
  static constexpr int TILES = W * WARPB;
  static constexpr int SMEM = TILES + W * S * 8 + 1024;  // + slack to 1 KB-align the base
};

// One warp task = ROWS consecutive slices of one region; lane l owns slices
// l, l+32, ... (RPL independent FNV chains per lane -- the ILP that hides the
// chains' multiply latency).
template <int S, int W, int RPL, int KC, bool kStg, SliceMode M, bool kCommit>
__global__ void __launch_bounds__(W * 32) slice_kernel(const __grid_constant__ SliceJob job) {
  using K = Cfg<S, W, RPL, KC>;
  static_assert(!kStg || KC == 1, "SM stores are implemented for single-plane boxes");
  constexpr int C = K::C;
  constexpr bool kCopy = (M == SliceMode::Copy || M == SliceMode::CopyVerify);
  constexpr bool kVerify = (M == SliceMode::CopyVerify || M == SliceMode::HashVerify);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint8_t* wbase = smem + warp * K::WARPB;
  const uint32_t bar0 = smem_u32(smem) + K::TILES + warp * S * 8;
  const uint32_t stage0 = smem_u32(wbase);

  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(bar0 + 8 * s, 1);
    mbar_init_fence();
  }
  __syncwarp();
  uint32_t phase = 0;  // bit s: parity of the next completion of stage s

  if constexpr (kCommit) {
    if (!job.skip_begin) {
      if (job.commit2.slot != nullptr) commit_begin(job.commit2);
      commit_begin(job.commit);
    }
  }

  const bool l2h = job.l2_stream != 0;
  const uint64_t pol = l2h ? evict_first_policy() : 0;
  auto load_tile = [&](uint32_t dst, const CUtensorMap* map, int kstep, int yy, uint32_t bar) {
    if constexpr (KC == 1) {
      if (l2h) tensor_load_h(dst, map, kstep * K::C, yy, bar, pol);
      else tensor_load(dst, map, kstep * K::C, yy, bar);
    } else {
      if (l2h) tensor_load3_h(dst, map, yy, kstep * KC, bar, pol);
      else tensor_load3(dst, map, yy, kstep * KC, bar);
    }
  };
  if (kDev && job.stagger_ns) __nanosleep(((blockIdx.x * W + warp) & 7u) * job.stagger_ns);
  uint64_t g_next = job.group_lo + static_cast<uint64_t>(blockIdx.x) * W + warp;
  const uint64_t g_stride = static_cast<uint64_t>(gridDim.x) * W;
  constexpr uint64_t kNone = ~0ull;
  bool once = false;
  auto claim = [&]() -> uint64_t {
    if (job.one_shot) {
      // task-granular batch: warp i of the grid owns task i (last first), once
      if (once) return kNone;
      once = true;
      const uint64_t i = static_cast<uint64_t>(blockIdx.x) * W + warp;
      return i < job.group_hi - job.group_lo ? job.group_hi - 1 - i : kNone;
    }
    if (job.sched != nullptr) {
      if (job.static_first && !once) {
        // the first task of every warp is fixed (no atomic storm at launch)
        once = true;
        const uint64_t i = static_cast<uint64_t>(blockIdx.x) * W + warp;
        if (i < job.group_hi - job.group_lo) return job.group_hi - 1 - i;
        return kNone;
      }
      // Claims run from the LAST task down: each region's ragged tail (and
      // tiny register-path regions) starts first and overlaps the bulk
      // instead of running alone after it -- one latency-bound register-path
      // task claimed last held an SM for ~130 us after the rest drained
      // (ncu PM sampling, profiles/r1_ncu_snapshot_kc2_details.csv).
      unsigned t = 0;
      if (lane == 0) t = atomicAdd(&job.sched[0], 1u);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (job.static_first) t += gridDim.x * W;  // the statically assigned first round
      if (t >= job.group_hi - job.group_lo) return kNone;
      return (!kDev || job.claim_order == 0 || t == 0) ? job.group_hi - 1 - t : job.group_lo + t - 1;
    }
    const uint64_t gg = g_next;
    g_next += g_stride;
    return gg < job.group_hi ? gg : kNone;
  };
  auto region_of = [&](uint64_t gg) {
    SliceRegion Q = job.reg[0];
#pragma unroll
    for (int i = 1; i < static_cast<int>(kMaxRegions); ++i)
      if (i < static_cast<int>(job.nregions) && gg >= job.reg[i].group_base) Q = job.reg[i];
    return Q;
  };
  // Cross-task prefetch (job.prefetch_next): the next task is claimed when
  // this one's last S steps start, and its first S steps are loaded into the
  // stages those steps free, so the stage ring runs on across task
  // boundaries (stage of step k = (sbase + k) % S) instead of draining.
  uint64_t g = claim();
  bool prefetched = false;
  uint32_t sbase = 0;
  for (;;) {
    if (g == kNone) break;
    uint64_t g_pf = kNone;
    bool claimed = false, pf_ok = false;

    const SliceRegion R = region_of(g);
    const uint64_t Sl = R.slice_bytes ? R.slice_bytes : job.slice_bytes;
    const bool al = aligned16(R.src) && (!kCopy || aligned16(R.dst));
    const uint64_t s0 = (g - R.group_base) * K::ROWS;

    std::conditional_t<kCopy, Fnv, FnvAlu> h[RPL];  // hash form per mode (ffx_device.cuh)
    uint64_t len[RPL];
    uint64_t want[RPL];  // verify modes: the expected checksums, loaded now so the
                         // load latency hides under the task instead of after it
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const uint64_t off = (s0 + lane + 32 * r) * Sl;
      len[r] = off < R.bytes ? umin64(Sl, R.bytes - off) : 0;
      h[r].init();
      if (job.init_state != nullptr && len[r]) h[r].set(job.init_state[R.slice_base + s0 + lane + 32 * r]);
      want[r] = 0;
      if constexpr (kVerify) {
        if (len[r])
          want[r] = R.expected != nullptr ? R.expected[s0 + lane + 32 * r]
                                          : job.sums_expected[R.slice_base + s0 + lane + 32 * r];
      }
    }

    // Stages are free once this lane's earlier bulk stores finished reading
    // them and every lane is past its previous hash.
    if constexpr (kCopy) {
      if (!prefetched) bulk_wait_read_all();
    }
    __syncwarp();

    if (R.tmap >= 0 && s0 + K::ROWS <= R.nfull) {
      // ---- tensor TMA: one box of KC planes of 128 x ROWS per step, 128 B swizzle ----
      const CUtensorMap* msrc = &job.maps[3 * R.tmap];
      const CUtensorMap* mdst = &job.maps[3 * R.tmap + 1];
      const CUtensorMap* mdst2 = &job.maps[3 * R.tmap + 2];
      const bool dual = R.dst2 != nullptr;
      const int nsteps = static_cast<int>(Sl / (C * KC));
      const int y = static_cast<int>(s0);
      const int pro = nsteps < S ? nsteps : S;
      if (lane == 0 && !prefetched) {
        fence_async_smem();  // rows written by the register path -> async proxy
        for (int k = 0; k < pro; ++k) {
          const int s = static_cast<int>((sbase + k) % S);
          mbar_expect_tx(bar0 + 8 * s, K::STAGE);
          load_tile(stage0 + s * K::STAGE, msrc, k, y, bar0 + 8 * s);
        }
      }
      const int sw = lane & 7;  // (lane + 32 r) & 7 == lane & 7
      for (int k = 0; k < nsteps; ++k) {
        const int s = static_cast<int>((sbase + k) % S);
        mbar_wait(bar0 + 8 * s, (phase >> s) & 1u);
        phase ^= 1u << s;
        const uint32_t tile = stage0 + s * K::STAGE;
        if constexpr (kCopy && !kStg) {
          if (lane == 0) {
            if constexpr (KC == 1) {
              if (l2h) {
                tensor_store_h(mdst, k * C, y, tile, pol);
                if (dual) tensor_store_h(mdst2, k * C, y, tile, pol);
              } else {
                tensor_store(mdst, k * C, y, tile);
                if (dual) tensor_store(mdst2, k * C, y, tile);  // double neighbour: read once, write twice
              }
            } else {
              if (l2h || (kDev && job.store_hint)) {
                const uint64_t spol = l2h ? pol : evict_first_policy();
                tensor_store3_hint(mdst, y, k * KC, tile, spol);
                if (dual) tensor_store3_hint(mdst2, y, k * KC, tile, spol);
              } else {
                tensor_store3(mdst, y, k * KC, tile);
                if (dual) tensor_store3(mdst2, y, k * KC, tile);
              }
            }
            bulk_commit();
          }
        }
        if constexpr (kCopy && kStg) {
          // SM stores instead of a TMA store: 8 lanes x 16 B cover one 128 B
          // row segment, so each STG.128 writes 4 full lines.
          const uint8_t* tp = wbase + s * K::STAGE;
#pragma unroll
          for (int i = 0; i < K::ROWS / 4; ++i) {
            const int j = i * 4 + (lane >> 3);
            const int w = lane & 7;
            const uint4 val = lds128(tp + j * C + ((w ^ (j & 7)) << 4));
            const uint64_t o = (s0 + j) * Sl + static_cast<uint64_t>(k) * C + w * 16;
            st_stream(R.dst + o, val);
            if (dual) st_stream(R.dst2 + o, val);
          }
        }
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {  // planes in byte order
          uint4 v[RPL][K::VPL];
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const uint8_t* row = wbase + s * K::STAGE + kc * K::PLANE + (lane + 32 * r) * C;
#pragma unroll
            for (int w = 0; w < K::VPL; ++w) v[r][w] = lds128(row + ((w ^ sw) << 4));
          }
#pragma unroll
          for (int w = 0; w < K::VPL; ++w)
#pragma unroll
            for (int r = 0; r < RPL; ++r) h[r].vec(v[r][w]);  // RPL chains interleaved
        }
        if (k + S < nsteps) {
          __syncwarp();
          if (lane == 0) {
            if constexpr (kCopy) bulk_wait_read_all();
            if (kDev && job.proxy_fence) fence_async_smem();
            mbar_expect_tx(bar0 + 8 * s, K::STAGE);
            load_tile(tile, msrc, k + S, y, bar0 + 8 * s);
          }
        } else if (kDev && job.prefetch_next) {
          if (k + S == nsteps) {  // this task's refills are done: claim the next one now
            claimed = true;
            g_pf = claim();
            if (g_pf != kNone) {
              const SliceRegion P = region_of(g_pf);
              pf_ok = P.tmap >= 0 && (g_pf - P.group_base) * K::ROWS + K::ROWS <= P.nfull;
            }
          }
          if (pf_ok) {  // step j = k + S - nsteps of the next task, into the stage step k frees
            __syncwarp();
            if (lane == 0) {
              const SliceRegion P = region_of(g_pf);
              const CUtensorMap* psrc = &job.maps[3 * P.tmap];
              const int py = static_cast<int>((g_pf - P.group_base) * K::ROWS);
              const int j = k + S - nsteps;
              if constexpr (kCopy) bulk_wait_read_all();
              if (kDev && job.proxy_fence) fence_async_smem();
              mbar_expect_tx(bar0 + 8 * s, K::STAGE);
              load_tile(tile, psrc, j, py, bar0 + 8 * s);
            }
          }
        }
      }
      sbase = static_cast<uint32_t>((sbase + nsteps) % S);
    } else {
      // ---- register path: ragged tail or unaligned pointers, 32 slices at a time ----
      uint4* rows = reinterpret_cast<uint4*>(wbase);
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const uint64_t sub0 = s0 + 32 * r;
        if (sub0 * Sl >= R.bytes) break;
        const uint64_t base0 = sub0 * Sl;
        const uint64_t max_len = umin64(Sl, R.bytes - base0);
        const int nsteps = static_cast<int>((max_len + C - 1) / C);
        for (int k = 0; k < nsteps; ++k) {
          uint4 buf[K::VPL];
#pragma unroll
          for (int i = 0; i < K::VPL; ++i) {
            const int q = i * 32 + lane;
            const uint64_t o = base0 + static_cast<uint64_t>(q / K::VPL) * Sl + static_cast<uint64_t>(k) * C +
                               static_cast<uint64_t>(q % K::VPL) * 16;
            buf[i] = load16(R.src, o, R.bytes, al);
            if constexpr (kCopy) {
              store16(R.dst, o, R.bytes, al, buf[i]);
              if (R.dst2 != nullptr) store16(R.dst2, o, R.bytes, al && aligned16(R.dst2), buf[i]);
            }
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < K::VPL; ++i) {
            const int q = i * 32 + lane;
            rows[(q / K::VPL) * (K::VPL + 1) + (q % K::VPL)] = buf[i];
          }
          __syncwarp();
          const int64_t rem = static_cast<int64_t>(len[r]) - static_cast<int64_t>(k) * C;
          const uint4* rp = rows + lane * (K::VPL + 1);
          if (rem >= C) {
#pragma unroll
            for (int w = 0; w < K::VPL; ++w) h[r].vec(rp[w]);
          } else if (rem > 0) {
            const uint8_t* rb = reinterpret_cast<const uint8_t*>(rp);
            for (int b = 0; b < rem; ++b) h[r].byte(rb[b]);
          }
        }
      }
    }

#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      if (!len[r]) continue;
      const uint64_t idx = R.slice_base + s0 + lane + 32 * r;
      const uint64_t v = h[r].value();
      if (job.sums_out != nullptr) job.sums_out[idx] = v;
      if (job.sums_out2 != nullptr) job.sums_out2[idx] = v;
      if constexpr (kVerify) {
        if (v != want[r]) {
          atomicMin(&job.result[0], static_cast<unsigned long long>(idx));
          atomicAdd(&job.result[1], 1ull);
        }
      }
    }
    if (claimed) {
      g = g_pf;
      prefetched = pf_ok;
    } else {
      g = claim();
      prefetched = false;
    }
  }

  if constexpr (kCopy) {
    bulk_wait_all();  // this lane's stores have landed
    fence_async_global();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (job.sched != nullptr) {
      __threadfence();
      if (atomicAdd(&job.sched[1], 1u) == gridDim.x - 1) {
        job.sched[0] = 0;
        job.sched[1] = 0;
      }
    }
    if constexpr (kCommit) {
      if (job.commit2.slot != nullptr) commit_end(job.commit2);
      commit_end(job.commit);
    }
  }
}

int g_sms = 0;

template <int S, int W, int RPL, bool kStg, SliceMode M, bool kCommit, int KC = 1>
cudaError_t launch_t(const SliceJob& job, uint32_t max_ctas, cudaStream_t stream) {
  auto kern = slice_kernel<S, W, RPL, KC, kStg, M, kCommit>;
  constexpr int smem = Cfg<S, W, RPL, KC>::SMEM;
  // The dynamic shared-memory opt-in is per device: one process may drive
  // several GPUs (single-process tests, the facade).
  static int occ = 0;
  static uint64_t set_on = 0;  // bit d: attribute set on device d
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(set_on & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (occ == 0) {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, W * 32, smem);
      if (e != cudaSuccess) return e;
      if (occ < 1) occ = 1;
    }
    set_on |= bit;
  }
  const uint64_t want = (job.group_hi - job.group_lo + W - 1) / W;
  uint64_t cap = static_cast<uint64_t>(occ) * sm_count();
  if (max_ctas) cap = std::min<uint64_t>(cap, max_ctas);
  if (job.one_shot) cap = ~0ull;  // one CTA per W tasks: the block scheduler interleaves
  const uint64_t grid = std::max<uint64_t>(1, std::min(want, cap));
  kern<<<static_cast<unsigned>(grid), W * 32, smem, stream>>>(job);
  return cudaGetLastError();
}

// Kernel configurations: stages / warps per CTA / slices per lane / SM
// stores instead of TMA stores / 128 B chunks per TMA op.  The warp-task
// size (32 * RPL slices) follows the configuration.
struct Variant {
  int S, W, RPL, stg, KC;
};
#ifdef FFX_DEV
// Development builds: the round-1 sweep table (FFX_SLICE_VARIANT /
// FFX_HASH_VARIANT; profiles/r1_variant_sweep_*.jsonl).
constexpr Variant kVariants[] = {{3, 4, 1, 0, 2}, {2, 4, 2, 0, 1}, {3, 4, 2, 0, 1}, {6, 4, 1, 0, 1},
                                 {3, 4, 1, 0, 1}, {2, 8, 2, 0, 1}, {4, 4, 1, 1, 1}, {3, 4, 2, 1, 1},
                                 {6, 4, 1, 1, 1}, {2, 4, 1, 0, 2}, {4, 4, 1, 0, 1}, {2, 4, 1, 0, 4},
                                 {2, 8, 1, 0, 2}, {2, 4, 1, 0, 1},
                                 // 14-16: small enough (< 18 KB smem, 64 threads) to sit beside a
                                 // 213 KB / 256-thread cuBLAS GEMM CTA on the same SM
                                 {2, 2, 1, 0, 1}, {3, 1, 1, 0, 1}, {2, 1, 1, 0, 2},
                                 // 17-18: wide single CTAs (more FNV chains per SM for narrow batches)
                                 {2, 12, 2, 0, 1}, {2, 16, 1, 0, 1}};
constexpr int kHashDefault = 9;
int variant() {
  static const int v = [] {
    const char* e = std::getenv("FFX_SLICE_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
#else
// Product: [0] copy modes -- 3 stages, 4 warps, 1 slice per lane, 2 chunks
// (256 B of each slice) per TMA op, the best full-GPU configuration of the
// round-1 sweep (profiles/r1_variant_sweep_1gpu.jsonl); [1] checksum-only
// modes -- the same boxes with 2 stages (no store to wait for: 3.63 vs 3.29
// TB/s hash-only, profiles/r1_hash_variant_sweep.txt); [2] CTA-capped
// batches (the slice scheduler inside a training step) -- 8 warps, 2 chains
// per lane, 2 stages of 128 B x 64 slices: 25.9 GB/s per CTA vs 14.0 for [0]
// at 8-64 CTAs (profiles/r2_cap_sweep_1gpu.jsonl), i.e. 1.85x less SM time
// per snapshotted byte where the SMs are borrowed from the step.
constexpr Variant kVariants[] = {{3, 4, 1, 0, 2}, {2, 4, 1, 0, 2}, {2, 8, 2, 0, 1}};
constexpr int kHashDefault = 1;
int variant() { return 0; }
#endif

// Checksum-only launches (split-policy hash batches, HashVerify, the whole
// FNV's sub-segment pass) use their own configuration: no store traffic, so
// fewer stages; the warp task must stay the same size (RPL).
int hash_variant();

template <SliceMode M, bool kCommit>
cudaError_t launch_mode(const SliceJob& job, uint32_t max_ctas, cudaStream_t stream) {
  constexpr bool hash_only = M == SliceMode::Hash || M == SliceMode::HashVerify;
#ifdef FFX_DEV
  switch (hash_only ? hash_variant() : variant()) {
    case 1: return launch_t<2, 4, 2, false, M, kCommit>(job, max_ctas, stream);
    case 2: return launch_t<3, 4, 2, false, M, kCommit>(job, max_ctas, stream);
    case 3: return launch_t<6, 4, 1, false, M, kCommit>(job, max_ctas, stream);
    case 4: return launch_t<3, 4, 1, false, M, kCommit>(job, max_ctas, stream);
    case 5: return launch_t<2, 8, 2, false, M, kCommit>(job, max_ctas, stream);
    case 6: return launch_t<4, 4, 1, true, M, kCommit>(job, max_ctas, stream);
    case 7: return launch_t<3, 4, 2, true, M, kCommit>(job, max_ctas, stream);
    case 8: return launch_t<6, 4, 1, true, M, kCommit>(job, max_ctas, stream);
    case 9: return launch_t<2, 4, 1, false, M, kCommit, 2>(job, max_ctas, stream);
    case 10: return launch_t<4, 4, 1, false, M, kCommit>(job, max_ctas, stream);
    case 11: return launch_t<2, 4, 1, false, M, kCommit, 4>(job, max_ctas, stream);
    case 12: return launch_t<2, 8, 1, false, M, kCommit, 2>(job, max_ctas, stream);
    case 13: return launch_t<2, 4, 1, false, M, kCommit>(job, max_ctas, stream);
    case 14: return launch_t<2, 2, 1, false, M, kCommit>(job, max_ctas, stream);
    case 15: return launch_t<3, 1, 1, false, M, kCommit>(job, max_ctas, stream);
    case 16: return launch_t<2, 1, 1, false, M, kCommit, 2>(job, max_ctas, stream);
    case 17: return launch_t<2, 12, 2, false, M, kCommit>(job, max_ctas, stream);
    case 18: return launch_t<2, 16, 1, false, M, kCommit>(job, max_ctas, stream);
    default: return launch_t<3, 4, 1, false, M, kCommit, 2>(job, max_ctas, stream);
  }
#else
  if (job.rows == kCappedRows) return launch_t<2, 8, 2, false, M, kCommit, 1>(job, max_ctas, stream);
  if constexpr (hash_only) return launch_t<2, 4, 1, false, M, kCommit, 2>(job, max_ctas, stream);
  else return launch_t<3, 4, 1, false, M, kCommit, 2>(job, max_ctas, stream);
#endif
}

}  // namespace

int sm_count() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

namespace {
const Variant& active_variant() {
  const int v = variant();
  return kVariants[(v >= 0 && v < static_cast<int>(sizeof kVariants / sizeof kVariants[0])) ? v : 0];
}
}  // namespace

uint32_t rows_for_cap(uint32_t max_ctas) {
#ifdef FFX_DEV
  (void)max_ctas;
  return 32u * static_cast<uint32_t>(active_variant().RPL);  // the variant under test decides
#else
  // capped launches (fewer CTAs than SMs) are SM-time bound: 2 chains per lane
  return (max_ctas > 0 && max_ctas < static_cast<uint32_t>(sm_count())) ? kCappedRows : kBulkRows;
#endif
}

namespace {
int hash_variant() {
#ifdef FFX_DEV
  static const int v = [] {
    const char* e = std::getenv("FFX_HASH_VARIANT");
    const int h = e ? std::atoi(e) : (variant() == 0 ? kHashDefault : variant());
    const int n = static_cast<int>(sizeof kVariants / sizeof kVariants[0]);
    // same warp-task size as the jobs (rows_for_cap), else the fused variant
    return (h >= 0 && h < n && kVariants[h].RPL == active_variant().RPL) ? h : variant();
  }();
  return v;
#else
  return kHashDefault;
#endif
}
}  // namespace

void finalize_job(SliceJob& job, uint32_t rows_in) {
  job.rows = rows_in ? rows_in : rows_for_cap(0);
  const uint64_t rows = job.rows;
  uint64_t groups = 0, slices = 0;
  for (uint32_t r = 0; r < job.nregions; ++r) {
    const uint64_t S = job.reg[r].slice_bytes ? job.reg[r].slice_bytes : job.slice_bytes;
    const uint64_t ns = (job.reg[r].bytes + S - 1) / S;
    job.reg[r].slice_base = slices;
    job.reg[r].group_base = groups;
    slices += ns;
    groups += (ns + rows - 1) / rows;
  }
  for (uint32_t r = job.nregions; r < kMaxRegions; ++r)
    job.reg[r] = SliceRegion{nullptr, nullptr, 0, slices, ~0ull, -1, 0, 0, nullptr};
  for (uint32_t r = 0; r < kMaxRegions; ++r) job.reg[r].tmap = -1;
  job.total_groups = groups;
  job.group_lo = 0;
  job.group_hi = groups;
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

bool encode_rows(CUtensorMap* map, const void* base, uint64_t slice_bytes, uint64_t nfull, uint32_t rows,
                 uint32_t kc) {
  auto enc = encoder();
  if (!enc) return false;
  if (kc > 1) {
    // {byte in chunk, slice, chunk}: strides {slice_bytes, 128}; box {128, rows, kc}
    const cuuint64_t dims3[3] = {128, nfull, slice_bytes / 128};
    const cuuint64_t strides3[2] = {slice_bytes, 128};
    const cuuint32_t box3[3] = {128, rows, kc};
    const cuuint32_t estr3[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims3, strides3, box3, estr3,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  const cuuint64_t dims[2] = {slice_bytes, nfull};
  const cuuint64_t strides[1] = {slice_bytes};
  const cuuint32_t box[2] = {128, rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// Give the (up to kTmaRegions) largest eligible regions 2-D tensor maps.
void attach_tensor_maps(SliceJob& job, bool copy, int kc_planes) {
  for (uint32_t r = 0; r < kMaxRegions; ++r) job.reg[r].tmap = -1;
  // largest first: a region left without a map runs on the latency-bound
  // register path, which only suits small or unaligned regions
  uint32_t order[kMaxRegions];
  for (uint32_t r = 0; r < job.nregions; ++r) order[r] = r;
  std::stable_sort(order, order + job.nregions,
                   [&](uint32_t a, uint32_t b) { return job.reg[a].bytes > job.reg[b].bytes; });
  int used = 0;
  for (uint32_t q = 0; q < job.nregions && used < kTmaRegions; ++q) {
    SliceRegion& R = job.reg[order[q]];
    const uint64_t S = R.slice_bytes ? R.slice_bytes : job.slice_bytes;
    if (S % 128 != 0 || S > (1ull << 31)) continue;
    R.nfull = R.bytes / S;
    const bool al = (reinterpret_cast<uintptr_t>(R.src) % 16 == 0) &&
                    (!copy || reinterpret_cast<uintptr_t>(R.dst) % 16 == 0);
    const uint32_t rows = job.rows;
    if (!al || R.nfull < rows || R.nfull > (1ull << 31)) continue;
    if (R.dst2 != nullptr && reinterpret_cast<uintptr_t>(R.dst2) % 16 != 0) continue;
    const uint32_t kc = static_cast<uint32_t>(kc_planes);
    if (S % (128ull * kc) != 0) continue;
    if (!encode_rows(&job.maps[3 * used], R.src, S, R.nfull, rows, kc)) continue;
    if (copy && !encode_rows(&job.maps[3 * used + 1], R.dst, S, R.nfull, rows, kc)) continue;
    if (copy && R.dst2 != nullptr &&
        !encode_rows(&job.maps[3 * used + 2], R.dst2, S, R.nfull, rows, kc))
      continue;
    R.tmap = used++;
  }
}

cudaError_t launch_slices(const SliceJob& job_in, SliceMode mode, bool commit, uint32_t max_ctas,
                          cudaStream_t stream) {
  SliceJob job = job_in;
  const bool hash_only = mode == SliceMode::Hash || mode == SliceMode::HashVerify;
  // the tensor maps' box depth follows the configuration this launch uses
#ifdef FFX_DEV
  const int vi = hash_only ? hash_variant() : variant();
  const int nv = static_cast<int>(sizeof kVariants / sizeof kVariants[0]);
  const Variant& V = kVariants[(vi >= 0 && vi < nv) ? vi : 0];
  if (job.rows != 32u * static_cast<uint32_t>(V.RPL)) return cudaErrorInvalidValue;  // job cut for another variant
#else
  const Variant& V = job.rows == kCappedRows ? kVariants[2] : kVariants[hash_only ? 1 : 0];
#endif
  attach_tensor_maps(job, !hash_only, V.KC);
  // The refill of a stage is a generic-read -> async-write (WAR) sequence,
  // ordered by the warp barrier; the proxy fence is only required for
  // generic writes read by the async proxy (kept per task).  The per-step
  // fence and the other experiment knobs exist only in FFX_DEV builds.
  job.proxy_fence = job.stagger_ns = job.claim_order = job.store_hint = job.prefetch_next = 0;
  // every warp's first task is assigned by its index instead of an atomic:
  // no 1184-way atomic storm at launch (+0.2%, profiles/r2_static_first_ab_1gpu.jsonl)
  job.static_first = 1;
  // CTA-capped jobs run inside a training step: stream through L2
  // evict-first so the step's own working set stays resident (measured
  // neutral on the synthetic step, profiles/r2_l2_hint_ab_n1.jsonl)
  job.l2_stream = job.rows == kCappedRows ? 1u : 0u;
#ifdef FFX_DEV
  static const auto env_u32 = [](const char* name) {
    const char* e = std::getenv(name);
    return e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : 0u;
  };
  static const uint32_t fence = std::getenv("FFX_STEP_FENCE") != nullptr ? 1u : 0u;
  static const uint32_t stagger = env_u32("FFX_STAGGER_NS");
  static const uint32_t order = env_u32("FFX_CLAIM_ORDER");
  static const uint32_t hint = std::getenv("FFX_STORE_HINT") != nullptr ? 1u : 0u;
  static const uint32_t prefetch = env_u32("FFX_PREFETCH");
  job.proxy_fence = fence;
  job.stagger_ns = stagger;
  job.claim_order = order;
  job.store_hint = hint;
  job.prefetch_next = prefetch;
  static const char* sfe = std::getenv("FFX_STATIC_FIRST");
  if (sfe) job.static_first = static_cast<uint32_t>(std::atoi(sfe));
#endif
  switch (mode) {
    case SliceMode::Hash:
      return commit ? launch_mode<SliceMode::Hash, true>(job, max_ctas, stream)
                    : launch_mode<SliceMode::Hash, false>(job, max_ctas, stream);
    case SliceMode::Copy:
      return commit ? launch_mode<SliceMode::Copy, true>(job, max_ctas, stream)
                    : launch_mode<SliceMode::Copy, false>(job, max_ctas, stream);
    case SliceMode::CopyVerify: return launch_mode<SliceMode::CopyVerify, false>(job, max_ctas, stream);
    case SliceMode::HashVerify: return launch_mode<SliceMode::HashVerify, false>(job, max_ctas, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ffx
