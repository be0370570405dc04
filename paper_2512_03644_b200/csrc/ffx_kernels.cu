// ffx_kernels.cu -- sm_100a kernels of the state-backup / recovery path.
//
//  slice_kernel   fused copy + per-slice FNV-1a-64 (+ verify, + slot commit):
//                 the snapshot kernel (local or NVLink-peer destination) and
//                 the recovery gather/verify kernel (peer source).
//  expand_kernel  evo::expand / evo::materialize (evolution.cpp:71-97).
//  check_kernel   evo::blob_is_sound (evolution.cpp:106-110).
//  fnv_spec_kernel + helpers: whole-buffer checksum64 (hash.cpp:102-110) by
//                 low-byte speculation and an affine combine.
//
// The path is HBM/NVLink-bound integer work: no tensor cores.  Global traffic
// is 16-byte vectorised and fully coalesced; the byte-serial FNV chains run
// one lane per slice out of a padded (conflict-free) shared-memory transpose.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "ffx_device.cuh"
#include "ffx_kernels.h"

namespace ffx {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 128;  // bytes of each slice staged per warp step

template <int C>
struct Stage {
  static constexpr int VPL = C / 16;   // 16-byte vectors per slice chunk (= per lane per step)
  static constexpr int ROW = VPL + 1;  // padded shared-memory row, in uint4
  static constexpr int SMEM = kWarps * 32 * ROW * 16;
};

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

// Load 16 bytes at base+o, zero beyond `bytes`; byte loads when unaligned or
// at a ragged tail.
__device__ __forceinline__ uint4 load16(const uint8_t* base, uint64_t o, uint64_t bytes, bool al) {
  if (al && o + 16 <= bytes) return ld_stream(base + o);
  uint4 v = make_uint4(0, 0, 0, 0);
  if (o < bytes) {
    uint32_t w[4] = {0, 0, 0, 0};
    const uint64_t n = bytes - o < 16 ? bytes - o : 16;
    for (uint64_t b = 0; b < n; ++b) w[b >> 2] |= static_cast<uint32_t>(base[o + b]) << (8 * (b & 3));
    v = make_uint4(w[0], w[1], w[2], w[3]);
  }
  return v;
}

__device__ __forceinline__ void store16(uint8_t* base, uint64_t o, uint64_t bytes, bool al,
                                        const uint4& v) {
  if (al && o + 16 <= bytes) {
    st_stream(base + o, v);
    return;
  }
  if (o < bytes) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    const uint64_t n = bytes - o < 16 ? bytes - o : 16;
    for (uint64_t b = 0; b < n; ++b) base[o + b] = static_cast<uint8_t>(w[b >> 2] >> (8 * (b & 3)));
  }
}

__device__ __forceinline__ void commit_begin(const SlotCommit& c) {
  if (threadIdx.x == 0) {
    volatile SlotMeta* m = reinterpret_cast<volatile SlotMeta*>(c.slot);
    m->magic = kSlotMagic;
    m->iteration = c.iteration;
    m->seq = c.seq;
    m->state = kSlotWriting;
    __threadfence_system();
  }
  __syncthreads();
}

__device__ __forceinline__ void commit_end(const SlotCommit& c) {
  __syncthreads();
  if (threadIdx.x != 0 || !c.finalize) return;
  __threadfence_system();
  const unsigned prev = atomicAdd(c.done, 1u);
  if (prev != gridDim.x - 1) return;
  __threadfence_system();
  volatile uint4* m = reinterpret_cast<volatile uint4*>(c.slot);
  for (int i = 1; i < static_cast<int>(kMetaBytes / 16); ++i) {
    const uint4 v = c.meta[i];
    m[i].x = v.x; m[i].y = v.y; m[i].z = v.z; m[i].w = v.w;
  }
  volatile uint4* h = reinterpret_cast<volatile uint4*>(c.slot + c.payload_off - 32);
  for (int i = 0; i < 2; ++i) {
    const uint4 v = c.snp1[i];
    h[i].x = v.x; h[i].y = v.y; h[i].z = v.z; h[i].w = v.w;
  }
  __threadfence_system();
  volatile SlotMeta* sm = reinterpret_cast<volatile SlotMeta*>(c.slot);
  sm->state = kSlotCommitted;
  __threadfence_system();
  *c.done = 0;
}

// One warp task = 32 consecutive slices of one region, one lane per slice.
// Per step the warp stages C bytes of each of its 32 slices: coalesced
// 16-byte loads (VPL per lane) -> optional 16-byte stores to the destination
// -> padded shared-memory rows -> each lane hashes its own row.  The next
// step's loads are issued before hashing, so HBM/NVLink latency overlaps the
// byte-serial FNV chains.
template <int C, SliceMode M, bool kCommit>
__global__ void __launch_bounds__(kThreads, 2) slice_kernel(const __grid_constant__ SliceJob job) {
  constexpr int VPL = Stage<C>::VPL;
  constexpr int ROW = Stage<C>::ROW;
  constexpr bool kCopy = (M == SliceMode::Copy || M == SliceMode::CopyVerify);
  constexpr bool kVerify = (M == SliceMode::CopyVerify || M == SliceMode::HashVerify);
  extern __shared__ uint4 smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint4* wsm = smem + warp * 32 * ROW;

  if constexpr (kCommit) commit_begin(job.commit);

  const uint64_t S = job.slice_bytes;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kWarps;
  for (uint64_t g = job.group_lo + static_cast<uint64_t>(blockIdx.x) * kWarps + warp;
       g < job.group_hi; g += stride) {
    SliceRegion R = job.reg[0];
#pragma unroll
    for (int i = 1; i < static_cast<int>(kMaxRegions); ++i)
      if (i < static_cast<int>(job.nregions) && g >= job.reg[i].group_base) R = job.reg[i];
    const bool al = aligned16(R.src) && (!kCopy || aligned16(R.dst));
    const uint64_t s0 = (g - R.group_base) * 32;
    const uint64_t base0 = s0 * S;
    const uint64_t my_off = base0 + static_cast<uint64_t>(lane) * S;
    const uint64_t my_len = my_off < R.bytes ? min(S, R.bytes - my_off) : 0;
    const uint64_t max_len = min(S, R.bytes - base0);
    const int nsteps = static_cast<int>((max_len + C - 1) / C);

    Fnv h;
    h.init();
    if (job.init_state != nullptr && my_len) h.set(job.init_state[R.slice_base + s0 + lane]);

    uint4 buf[VPL];
    auto voff = [&](int i, int k) -> uint64_t {
      const int q = i * 32 + lane;
      return base0 + static_cast<uint64_t>(q / VPL) * S + static_cast<uint64_t>(k) * C +
             static_cast<uint64_t>(q % VPL) * 16;
    };
    // Fast path: the whole task is 32 full, aligned slices.
    const bool full = al && base0 + 32 * S <= R.bytes;
    auto load_step = [&](int k) {
      if (full) {
#pragma unroll
        for (int i = 0; i < VPL; ++i) buf[i] = ld_stream(R.src + voff(i, k));
      } else {
#pragma unroll
        for (int i = 0; i < VPL; ++i) buf[i] = load16(R.src, voff(i, k), R.bytes, al);
      }
    };
    load_step(0);

    for (int k = 0; k < nsteps; ++k) {
      __syncwarp();
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int q = i * 32 + lane;
        wsm[(q / VPL) * ROW + (q % VPL)] = buf[i];
      }
      if constexpr (kCopy) {
        if (full) {
#pragma unroll
          for (int i = 0; i < VPL; ++i) st_stream(R.dst + voff(i, k), buf[i]);
        } else {
#pragma unroll
          for (int i = 0; i < VPL; ++i) store16(R.dst, voff(i, k), R.bytes, al, buf[i]);
        }
      }
      __syncwarp();
      if (k + 1 < nsteps) load_step(k + 1);
      const int64_t rem = static_cast<int64_t>(my_len) - static_cast<int64_t>(k) * C;
      if (rem >= C) {
#pragma unroll
        for (int w = 0; w < VPL; ++w) h.vec(wsm[lane * ROW + w]);
      } else if (rem > 0) {
        const uint8_t* row = reinterpret_cast<const uint8_t*>(wsm + lane * ROW);
        for (int b = 0; b < rem; ++b) h.byte(row[b]);
      }
    }
    if (my_len) {
      const uint64_t idx = R.slice_base + s0 + lane;
      const uint64_t v = h.value();
      if (job.sums_out != nullptr) job.sums_out[idx] = v;
      if constexpr (kVerify) {
        if (v != job.sums_expected[idx]) {
          atomicMin(&job.result[0], static_cast<unsigned long long>(idx));
          atomicAdd(&job.result[1], 1ull);
        }
      }
    }
  }

  if constexpr (kCommit) commit_end(job.commit);
}

int g_sms = 0;

template <int C, SliceMode M, bool kCommit>
cudaError_t launch_t(const SliceJob& job, uint32_t max_ctas, cudaStream_t stream) {
  auto kern = slice_kernel<C, M, kCommit>;
  constexpr int smem = Stage<C>::SMEM;
  static int occ = 0;
  if (occ == 0) {
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  uint64_t want = (job.group_hi - job.group_lo + kWarps - 1) / kWarps;
  uint64_t cap = static_cast<uint64_t>(occ) * sm_count();
  if (max_ctas) cap = std::min<uint64_t>(cap, max_ctas);
  uint64_t grid = std::max<uint64_t>(1, std::min(want, cap));
  kern<<<static_cast<unsigned>(grid), kThreads, smem, stream>>>(job);
  return cudaGetLastError();
}

// ---- synthetic state ----------------------------------------------------------

// Vector t covers bytes [16t, 16t+16).  With word_base in {0, 32} a vector is
// either all prefix or exactly words 2u, 2u+1 (u = (16t - word_base) / 16).
__global__ void expand_kernel(uint8_t* dst, uint64_t fold, uint64_t bytes, uint64_t word_base,
                              uint4 p0, uint4 p1) {
  const uint64_t nvec = (bytes + 15) / 16;
  const bool al = aligned16(dst);
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < nvec;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t o = 16 * t;
    uint4 v;
    if (o < word_base) {
      v = (o == 0) ? p0 : p1;
    } else {
      const uint64_t w = (o - word_base) / 8;
      const uint64_t a = mix64(fold + (w + 1) * kGolden);
      const uint64_t b = mix64(fold + (w + 2) * kGolden);
      v = make_uint4(static_cast<uint32_t>(a), static_cast<uint32_t>(a >> 32),
                     static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32));
    }
    store16(dst, o, bytes, al, v);
  }
}

__global__ void check_kernel(const uint8_t* blob, uint64_t bytes, unsigned long long* result) {
  uint64_t fold = 0;
  for (int i = 7; i >= 0; --i) fold = (fold << 8) | blob[i];
  const uint64_t nvec = (bytes + 15) / 16;
  const bool al = aligned16(blob);
  for (uint64_t t = 2 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < nvec;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t o = 16 * t;
    const uint64_t w = (o - 32) / 8;
    const uint64_t a = mix64(fold + (w + 1) * kGolden);
    const uint64_t b = mix64(fold + (w + 2) * kGolden);
    const uint4 got = load16(blob, o, bytes, al);
    const uint32_t want[4] = {static_cast<uint32_t>(a), static_cast<uint32_t>(a >> 32),
                              static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32)};
    const uint32_t have[4] = {got.x, got.y, got.z, got.w};
    const uint64_t n = bytes - o < 16 ? bytes - o : 16;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t diff = want[i] ^ have[i];
      const int64_t valid = static_cast<int64_t>(n) - 4 * i;
      if (valid <= 0) diff = 0;
      else if (valid < 4) diff &= (1u << (8 * valid)) - 1u;
      if (diff) {
        atomicMin(result, static_cast<unsigned long long>(o + 4 * i + (__ffs(diff) - 1) / 8));
        break;
      }
    }
  }
}

// ---- whole-buffer FNV-1a-64 ---------------------------------------------------
//
// The low byte l of the FNV state evolves autonomously:
//   l' = ((l ^ b) * 0xB3) mod 256            (0xB3 = FNV prime mod 256)
// and h_{i+1} = h_i * P + ((l_i ^ b_i) - l_i) * P, so once the low-byte
// trajectory is known each sub-segment is an affine map h -> A*h + B.
//  phase 1  fnv_spec_kernel: per segment (K sub-segments), all 256 start
//           values of l simulated in parallel (two per 32-bit lane), recording
//           the state at every sub-segment end -> T[sub][start].
//  phase 2  fnv_walk_kernel: chain segment start states l through T.
//  phase 3  fnv_init_kernel + slice_kernel(Hash, init_state=l_sub):
//           F_sub = FNV of the sub-segment started from h = l_sub.
//  phase 4  fnv_combine_kernel: h = fold_sub (h - l_sub) * P^len_sub + F_sub.

constexpr int kSpecK = 16;  // sub-segments per segment

__global__ void fnv_spec_kernel(const uint8_t* data, uint64_t len, uint64_t Ls, uint64_t nsub,
                                uint8_t* T) {
  const uint64_t gt = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t seg = gt / 16;
  const int t = static_cast<int>(gt % 16);
  const uint64_t sub0 = seg * kSpecK;
  if (sub0 >= nsub) return;
  const uint64_t sub1 = min(sub0 + kSpecK, nsub);
  uint32_t x[8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
    x[r] = static_cast<uint32_t>(t * 16 + 2 * r) | (static_cast<uint32_t>(t * 16 + 2 * r + 1) << 16);
  const bool al = aligned16(data);
  for (uint64_t u = sub0; u < sub1; ++u) {
    const uint64_t b0 = u * Ls;
    const uint64_t b1 = min(b0 + Ls, len);
    for (uint64_t o = b0; o < b1; o += 16) {
      const uint4 v = load16(data, o, b1, al);
      const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
      const int n = static_cast<int>(umin64(16, b1 - o));
      if (n == 16) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t bb = __byte_perm(w4[q >> 2], 0u, 0x4040 + 0x0101 * (q & 3));
#pragma unroll
          for (int r = 0; r < 8; ++r) x[r] = ((x[r] & 0x00FF00FFu) ^ bb) * 0xB3u;
        }
      } else {
        for (int q = 0; q < n; ++q) {
          const uint32_t bb = __byte_perm(w4[q >> 2], 0u, 0x4040 + 0x0101 * (q & 3));
#pragma unroll
          for (int r = 0; r < 8; ++r) x[r] = ((x[r] & 0x00FF00FFu) ^ bb) * 0xB3u;
        }
      }
    }
    uint32_t out[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t a = x[2 * r], b = x[2 * r + 1];
      out[r] = (a & 0xffu) | (((a >> 16) & 0xffu) << 8) | ((b & 0xffu) << 16) | (((b >> 16) & 0xffu) << 24);
    }
    reinterpret_cast<uint4*>(T + u * 256)[t] = make_uint4(out[0], out[1], out[2], out[3]);
  }
}

// One CTA: walk segment ends; lam_seg[s] = low byte at segment s start.
__global__ void fnv_walk_kernel(const uint8_t* T, uint64_t nsub, uint64_t nseg, uint32_t l0,
                                uint8_t* lam_seg) {
  __shared__ uint4 tab[32][16];  // 32 segment-end tables
  uint32_t l = l0;
  for (uint64_t s0 = 0; s0 < nseg; s0 += 32) {
    const uint64_t cnt = umin64(32, nseg - s0);
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < cnt * 16; i += blockDim.x) {
      const uint64_t s = s0 + i / 16;
      const uint64_t last = umin64(s * kSpecK + kSpecK, nsub) - 1;
      tab[i / 16][i % 16] = reinterpret_cast<const uint4*>(T + last * 256)[i % 16];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (uint64_t i = 0; i < cnt; ++i) {
        lam_seg[s0 + i] = static_cast<uint8_t>(l);
        l = reinterpret_cast<const uint8_t*>(tab[i])[l];
      }
    }
  }
}

__global__ void fnv_init_kernel(const uint8_t* T, const uint8_t* lam_seg, uint64_t nsub,
                                uint64_t* init) {
  for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; u < nsub;
       u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t seg = u / kSpecK;
    const uint32_t ls = lam_seg[seg];
    init[u] = (u % kSpecK == 0) ? ls : T[(u - 1) * 256 + ls];
  }
}

// One CTA of 1024 threads folds the affine maps of all sub-segments in order.
__global__ void fnv_combine_kernel(const uint64_t* init, const uint64_t* F, uint64_t nsub,
                                   uint64_t A_full, uint64_t A_last, uint64_t h0, uint64_t* out) {
  __shared__ uint64_t sa[1024], sb[1024];
  const uint64_t per = (nsub + blockDim.x - 1) / blockDim.x;
  const uint64_t u0 = threadIdx.x * per;
  const uint64_t u1 = min(u0 + per, nsub);
  uint64_t A = 1, B = 0;  // composite map h -> A*h + B
  for (uint64_t u = u0; u < u1; ++u) {
    const uint64_t a = (u + 1 == nsub) ? A_last : A_full;
    const uint64_t b = F[u] - init[u] * a;
    A = a * A;
    B = a * B + b;
  }
  sa[threadIdx.x] = A;
  sb[threadIdx.x] = B;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t h = h0;
    for (unsigned i = 0; i < blockDim.x; ++i) h = sa[i] * h + sb[i];
    *out = h;
  }
}

uint64_t pow_mod64(uint64_t base, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r *= base;
    base *= base;
    e >>= 1;
  }
  return r;
}

__global__ void fill_kernel(uint8_t* dst, uint64_t bytes, uint32_t pattern) {
  const bool al = aligned16(dst);
  const uint4 v = make_uint4(pattern, pattern, pattern, pattern);
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t * 16 < bytes;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    store16(dst, 16 * t, bytes, al, v);
}

__global__ void xor_byte_kernel(uint8_t* dst, uint8_t mask) { *dst ^= mask; }

unsigned grid_for(uint64_t work_items, int threads) {
  const uint64_t want = (work_items + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(sm_count()) * 8;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min(want, cap)));
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

void finalize_job(SliceJob& job) {
  uint64_t groups = 0, slices = 0;
  for (uint32_t r = 0; r < job.nregions; ++r) {
    const uint64_t ns = (job.reg[r].bytes + job.slice_bytes - 1) / job.slice_bytes;
    job.reg[r].slice_base = slices;
    job.reg[r].group_base = groups;
    slices += ns;
    groups += (ns + 31) / 32;
  }
  for (uint32_t r = job.nregions; r < kMaxRegions; ++r) {
    job.reg[r] = SliceRegion{nullptr, nullptr, 0, slices, ~0ull};
  }
  job.total_groups = groups;
  job.group_lo = 0;
  job.group_hi = groups;
}

cudaError_t launch_slices(const SliceJob& job, SliceMode mode, bool commit, uint32_t max_ctas,
                          cudaStream_t stream) {
  switch (mode) {
    case SliceMode::Hash:
      return launch_t<kChunk, SliceMode::Hash, false>(job, max_ctas, stream);
    case SliceMode::Copy:
      return commit ? launch_t<kChunk, SliceMode::Copy, true>(job, max_ctas, stream)
                    : launch_t<kChunk, SliceMode::Copy, false>(job, max_ctas, stream);
    case SliceMode::CopyVerify:
      return launch_t<kChunk, SliceMode::CopyVerify, false>(job, max_ctas, stream);
    case SliceMode::HashVerify:
      return launch_t<kChunk, SliceMode::HashVerify, false>(job, max_ctas, stream);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_expand(uint8_t* dst, uint64_t fold, uint64_t bytes, const uint8_t* prefix32,
                          cudaStream_t stream) {
  if (bytes == 0) return cudaSuccess;
  uint4 p[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
  if (prefix32) memcpy(p, prefix32, 32);
  expand_kernel<<<grid_for((bytes + 15) / 16, 256), 256, 0, stream>>>(dst, fold, bytes,
                                                                     prefix32 ? 32 : 0, p[0], p[1]);
  return cudaGetLastError();
}

cudaError_t launch_blob_check(const uint8_t* blob, uint64_t bytes, unsigned long long* result,
                              cudaStream_t stream) {
  if (bytes <= 32) return cudaSuccess;
  check_kernel<<<grid_for((bytes + 15) / 16, 256), 256, 0, stream>>>(blob, bytes, result);
  return cudaGetLastError();
}

cudaError_t whole_fnv(const uint8_t* data, uint64_t len, uint64_t h0, uint64_t* out,
                      cudaStream_t stream) {
  if (len == 0) {
    *out = h0;
    return cudaSuccess;
  }
  // Sub-segment length: >= 4 KiB, sized for ~128K independent chains.
  uint64_t Ls = std::max<uint64_t>(4096, align_up((len + 131071) / 131072, 256));
  const uint64_t nsub = (len + Ls - 1) / Ls;
  const uint64_t nseg = (nsub + kSpecK - 1) / kSpecK;
  const uint64_t last_len = len - (nsub - 1) * Ls;

  uint8_t* scratch = nullptr;
  const uint64_t offT = 0, offLam = align_up(nsub * 256, 256),
                 offInit = offLam + align_up(nseg, 256), offF = offInit + align_up(nsub * 8, 256),
                 offOut = offF + align_up(nsub * 8, 256), total = offOut + 256;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), total, stream);
  if (e != cudaSuccess) return e;
  uint8_t* T = scratch + offT;
  uint8_t* lam = scratch + offLam;
  uint64_t* init = reinterpret_cast<uint64_t*>(scratch + offInit);
  uint64_t* F = reinterpret_cast<uint64_t*>(scratch + offF);
  uint64_t* dout = reinterpret_cast<uint64_t*>(scratch + offOut);

  const uint64_t spec_threads = nseg * 16;
  fnv_spec_kernel<<<static_cast<unsigned>((spec_threads + 255) / 256), 256, 0, stream>>>(
      data, len, Ls, nsub, T);
  fnv_walk_kernel<<<1, 512, 0, stream>>>(T, nsub, nseg, static_cast<uint32_t>(h0 & 0xff), lam);
  fnv_init_kernel<<<grid_for(nsub, 256), 256, 0, stream>>>(T, lam, nsub, init);
  // The high bits of the true state enter only through the affine combine, so
  // each sub-segment starts from its low byte alone.
  SliceJob job{};
  job.nregions = 1;
  job.reg[0] = SliceRegion{data, nullptr, len, 0, 0};
  job.slice_bytes = Ls;
  job.sums_out = F;
  job.init_state = init;
  finalize_job(job);
  e = launch_slices(job, SliceMode::Hash, false, 0, stream);
  if (e != cudaSuccess) return e;
  fnv_combine_kernel<<<1, 1024, 0, stream>>>(init, F, nsub, pow_mod64(kFnvPrime, Ls),
                                             pow_mod64(kFnvPrime, last_len), h0, dout);
  e = cudaMemcpyAsync(out, dout, 8, cudaMemcpyDeviceToHost, stream);
  if (e != cudaSuccess) return e;
  e = cudaFreeAsync(scratch, stream);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(stream);
}

cudaError_t launch_fill(uint8_t* dst, uint64_t bytes, uint32_t pattern, cudaStream_t stream) {
  if (bytes == 0) return cudaSuccess;
  fill_kernel<<<grid_for((bytes + 15) / 16, 256), 256, 0, stream>>>(dst, bytes, pattern);
  return cudaGetLastError();
}

cudaError_t launch_xor_byte(uint8_t* dst, uint8_t mask, cudaStream_t stream) {
  xor_byte_kernel<<<1, 1, 0, stream>>>(dst, mask);
  return cudaGetLastError();
}

}  // namespace ffx
