// ffx_kernels.cu -- sm_100a kernels of the state-backup / recovery path.
//
//  (the snapshot / recovery slice kernel lives in ffx_slice.cu)
//  expand_kernel  evo::expand / evo::materialize (evolution.cpp:71-97).
//  check_kernel   evo::blob_is_sound (evolution.cpp:106-110).
//  fnv_spec_kernel + helpers: whole-buffer checksum64 (hash.cpp:102-110) by
//                 low-byte speculation and an affine combine.
//
// HBM-bound integer work: 16-byte vectorised, coalesced, grid-stride.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "ffx_device.cuh"
#include "ffx_kernels.h"

namespace ffx {

namespace {

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

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

// ---- synthetic state ----------------------------------------------------------

// Vector t covers bytes [16t, 16t+16).  With word_base in {0, 32} a vector is
// either all prefix or exactly words 2u, 2u+1 (u = (16t - word_base) / 16).
__global__ void expand_kernel(uint8_t* dst, uint64_t fold, uint64_t bytes, uint64_t word_base,
                              uint4 p0, uint4 p1) {
  // Vector t (bytes [16t, 16t+16)) holds words w, w+1 with w = 2t - word_base/8,
  // i.e. mix64(fold + (w+1)G), mix64(fold + (w+2)G): the argument advances
  // by 2G per vector, so by a constant per grid-stride step (mod 2^64).
  const uint64_t nvec = (bytes + 15) / 16;
  const uint64_t nfull = bytes / 16;
  const bool al = aligned16(dst);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t t_first = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  uint64_t s = fold + (2 * t_first - word_base / 8 + 1) * kGolden;
  const uint64_t dS = 2 * stride * kGolden;
  for (uint64_t t = t_first; t < nvec; t += stride, s += dS) {
    const uint64_t o = 16 * t;
    uint4 v;
    if (o < word_base) {
      v = (o == 0) ? p0 : p1;
    } else {
      const uint64_t a = mix64(s);
      const uint64_t b = mix64(s + kGolden);
      v = make_uint4(static_cast<uint32_t>(a), static_cast<uint32_t>(a >> 32),
                     static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32));
    }
    if (al && t < nfull) st_stream(dst + o, v);
    else store16(dst, o, bytes, al, v);
  }
}

// blob_is_sound, one 16-byte vector (bytes past `bytes` ignored).
__device__ __forceinline__ void check_vec(uint64_t fold, uint64_t o, uint64_t bytes, const uint4& got,
                                          unsigned long long* result) {
  const uint64_t w = (o - 32) / 8;
  const uint64_t a = mix64(fold + (w + 1) * kGolden);
  const uint64_t b = mix64(fold + (w + 2) * kGolden);
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

constexpr int kCheckUnroll = 4;  // 16-byte loads in flight per thread (read-only stream)

// blob_is_sound over [32, bytes): vector t (bytes [16t, 16t+16)) must equal
// words 2t-4 and 2t-3 of the expansion, i.e. mix64(fold + (2t-3)G) and
// mix64(fold + (2t-2)G) (evolution.cpp:71-84).  The mix64 arguments advance by
// a constant per grid-stride step, so no 64-bit multiply by the index; whole
// aligned vectors compare as two 64-bit words, the byte-exact search for the
// first difference only runs on a mismatch or the ragged tail.
__global__ void check_kernel(const uint8_t* blob, uint64_t bytes, unsigned long long* result) {
  __shared__ uint64_t s_fold;
  if (threadIdx.x == 0) {
    uint64_t f = 0;
    for (int i = 7; i >= 0; --i) f = (f << 8) | blob[i];
    s_fold = f;
  }
  __syncthreads();
  const uint64_t fold = s_fold;
  const uint64_t nvec = (bytes + 15) / 16;
  const uint64_t nfull = bytes / 16;
  const bool al = aligned16(blob);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t t_first = 2 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t dS = 2 * stride * kGolden;  // mix64-argument step between u and u+1
  uint64_t s0 = fold + (2 * t_first - 3) * kGolden;
  for (uint64_t t0 = t_first; t0 < nvec; t0 += kCheckUnroll * stride, s0 += kCheckUnroll * dS) {
    uint4 got[kCheckUnroll];
#pragma unroll
    for (int u = 0; u < kCheckUnroll; ++u) {  // issue every load before any compare
      const uint64_t t = t0 + u * stride;
      got[u] = (al && t < nfull) ? ld_stream(blob + 16 * t)
                                 : (t < nvec ? load16(blob, 16 * t, bytes, al) : make_uint4(0, 0, 0, 0));
    }
#pragma unroll
    for (int u = 0; u < kCheckUnroll; ++u) {
      const uint64_t t = t0 + u * stride;
      if (t >= nvec) break;
      const uint64_t s = s0 + u * dS;
      const uint64_t a = mix64(s), b = mix64(s + kGolden);
      const uint64_t ga = (static_cast<uint64_t>(got[u].y) << 32) | got[u].x;
      const uint64_t gb = (static_cast<uint64_t>(got[u].w) << 32) | got[u].z;
      if (t < nfull && ga == a && gb == b) continue;
      check_vec(fold, 16 * t, bytes, got[u], result);  // mismatch or ragged tail: find the byte
    }
  }
}

// ---- whole-buffer FNV-1a-64 ---------------------------------------------------
//
// The low byte l of the FNV state evolves autonomously:
//   l' = ((l ^ b) * 0xB3) mod 256            (0xB3 = FNV prime mod 256)
// and h_{i+1} = h_i * P + ((l_i ^ b_i) - l_i) * P, so once the low-byte
// trajectory is known each sub-segment is an affine map h -> A*h + B.
//  phase 1  fnv_spec_kernel: per segment (K sub-segments), start values
//           l = 0..63 simulated in parallel (two per 32-bit lane), recording
//           the state at every sub-segment end -> T[sub][start] and the
//           running parity of bit 6 of the data.  Bit 7 never feeds lower
//           bits: x ^ 0x80 = x + 128 and 128 * 0xB3 = 128 (mod 256), so the
//           trajectory from l ^ 0x80 is the one from l with bit 7 flipped at
//           every step.  Bit 6 only feeds bit 7: from l ^ 0x40 the trajectory
//           keeps bits 0-5, complements bit 6, and flips bit 7 whenever
//           bit6(l_i ^ b_i) == bit6(l_{i+1}); those flips telescope to
//           (n & 1) ^ bit6(l_0) ^ bit6(l_n) ^ parity(bit 6 of the n bytes), so
//           64 simulated starts give all 256 (spec_lookup): a quarter of the
//           naive speculation.
//  phase 2  fnv_walk_kernel: chain segment start states l through T.
//  phase 3  fnv_init_kernel + slice_kernel(Hash, init_state=l_sub):
//           F_sub = FNV of the sub-segment started from h = l_sub.
//  phase 4  fnv_combine_kernel: h = fold_sub (h - l_sub) * P^len_sub + F_sub.

constexpr int kSpecK = 8;        // sub-segments per segment
constexpr int kSpecRegs = 8;     // packed registers per thread: 2 start values each (4 threads: 7.5 ms; 8: 9.1)
constexpr int kSpecThreads = 64 / (2 * kSpecRegs);  // threads per segment (64 simulated starts)
constexpr int kSpecTab = 64;     // table entries per sub-segment (bits 6 and 7 derived)

// Full end state for start l from the 64-entry table of starts l & 63:
// bit 7 is symmetric (see above); for bit 6 the trajectory from l0 ^ 0x40
// is that from l0 with bit 6 complemented and bit 7 flipped d times, and the
// flips telescope to d = (n & 1) ^ bit6(end state) ^ (parity of bit 6 over
// the n data bytes) -- so 64 simulated starts give all 256.
__device__ __forceinline__ uint32_t spec_lookup(const uint8_t* Tu, uint32_t odd, uint32_t l) {
  const uint32_t a = Tu[l & 63u];
  uint32_t r = a;
  if (l & 0x40u) r ^= 0x40u ^ (((odd ^ (a >> 6)) & 1u) << 7);
  return r ^ (l & 0x80u);
}

// bytes from the start of sub-segment u's segment through the end of u
__device__ __forceinline__ uint64_t spec_span(uint64_t u, uint64_t Ls, uint64_t len) {
  const uint64_t seg0 = (u / kSpecK) * kSpecK * Ls;
  return umin64((u + 1) * Ls, len) - seg0;
}

__global__ void fnv_spec_kernel(const uint8_t* data, uint64_t len, uint64_t Ls, uint64_t nsub,
                                uint8_t* T, uint8_t* P) {
  const uint64_t gt = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t seg = gt / kSpecThreads;
  const int t = static_cast<int>(gt % kSpecThreads);
  const uint64_t sub0 = seg * kSpecK;
  if (sub0 >= nsub) return;
  const uint64_t sub1 = min(sub0 + kSpecK, nsub);
  constexpr int R = kSpecRegs;
  uint32_t x[R];
#pragma unroll
  for (int r = 0; r < R; ++r)
    x[r] = static_cast<uint32_t>(t * 2 * R + 2 * r) | (static_cast<uint32_t>(t * 2 * R + 2 * r + 1) << 16);
  const bool al = aligned16(data);
  uint32_t par = 0;  // thread 0: running parity of bit 6 of the data bytes (bits 6, 14, 22, 30)
  for (uint64_t u = sub0; u < sub1; ++u) {
    const uint64_t b0 = u * Ls;
    const uint64_t b1 = min(b0 + Ls, len);
    for (uint64_t o = b0; o < b1; o += 16) {
      const uint4 v = load16(data, o, b1, al);  // zero-filled past b1: parity unaffected
      if (t == 0) par ^= v.x ^ v.y ^ v.z ^ v.w;
      const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
      const int n = static_cast<int>(umin64(16, b1 - o));
      if (n == 16) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t bb = __byte_perm(w4[q >> 2], 0u, 0x4040 + 0x0101 * (q & 3));
#pragma unroll
          for (int r = 0; r < R; ++r) x[r] = ((x[r] & 0x00FF00FFu) ^ bb) * 0xB3u;
        }
      } else {
        for (int q = 0; q < n; ++q) {
          const uint32_t bb = __byte_perm(w4[q >> 2], 0u, 0x4040 + 0x0101 * (q & 3));
#pragma unroll
          for (int r = 0; r < R; ++r) x[r] = ((x[r] & 0x00FF00FFu) ^ bb) * 0xB3u;
        }
      }
    }
    uint32_t out[R / 2];
#pragma unroll
    for (int r = 0; r < R / 2; ++r) {
      const uint32_t a = x[2 * r], b = x[2 * r + 1];
      out[r] = (a & 0xffu) | (((a >> 16) & 0xffu) << 8) | ((b & 0xffu) << 16) | (((b >> 16) & 0xffu) << 24);
    }
#pragma unroll
    for (int r = 0; r < R / 2; ++r) reinterpret_cast<uint32_t*>(T + u * kSpecTab)[t * (R / 2) + r] = out[r];
    // P[u] = (n & 1) ^ parity of bit 6 through the end of u: the "odd" input of spec_lookup
    if (t == 0) P[u] = static_cast<uint8_t>((__popc(par & 0x40404040u) ^ spec_span(u, Ls, len)) & 1u);
  }
}

// One CTA: walk segment ends; lam_seg[s] = low byte at segment s start.
__global__ void fnv_walk_kernel(const uint8_t* T, const uint8_t* P, uint64_t nsub, uint64_t nseg, uint32_t l0,
                                uint8_t* lam_seg) {
  constexpr int kV = kSpecTab / 16;  // uint4 per table
  __shared__ uint4 tab[128][kV];     // 128 segment-end tables
  __shared__ uint8_t odd[128];
  uint32_t l = l0;
  for (uint64_t s0 = 0; s0 < nseg; s0 += 128) {
    const uint64_t cnt = umin64(128, nseg - s0);
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < cnt * kV; i += blockDim.x) {
      const uint64_t s = s0 + i / kV;
      const uint64_t last = umin64(s * kSpecK + kSpecK, nsub) - 1;
      tab[i / kV][i % kV] = reinterpret_cast<const uint4*>(T + last * kSpecTab)[i % kV];
      if (i % kV == 0) odd[i / kV] = P[last];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (uint64_t i = 0; i < cnt; ++i) {
        lam_seg[s0 + i] = static_cast<uint8_t>(l);
        l = spec_lookup(reinterpret_cast<const uint8_t*>(tab[i]), odd[i], l);
      }
    }
  }
}

__global__ void fnv_init_kernel(const uint8_t* T, const uint8_t* P, const uint8_t* lam_seg, uint64_t nsub,
                                uint64_t* init) {
  for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; u < nsub;
       u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t seg = u / kSpecK;
    const uint32_t ls = lam_seg[seg];
    init[u] = (u % kSpecK == 0) ? ls : spec_lookup(T + (u - 1) * kSpecTab, P[u - 1], ls);
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

// ---- data loader: synthetic samples and their fold ----------------------------

// Word w of sample i is mix64(fold_i + (w+1) G) (expand, evolution.cpp:71-97);
// samples are packed back to back, so a sample need not start 8-aligned:
// aligned full words go out as one 8-byte store, the rest byte by byte.
__global__ void items_kernel(uint8_t* dst, const uint64_t* folds, uint32_t count, uint32_t sample_bytes) {
  const uint64_t wps = (sample_bytes + 7) / 8;  // words per sample
  const uint64_t total = wps * count;
  for (uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = g / wps, w = g % wps;
    const uint64_t v = mix64(folds[i] + (w + 1) * kGolden);
    const uint64_t o = i * sample_bytes + 8 * w;
    const uint32_t n = static_cast<uint32_t>(umin64(8, sample_bytes - 8 * w));
    uint8_t* p = dst + o;
    if (n == 8 && (reinterpret_cast<uintptr_t>(p) & 7u) == 0) {
      *reinterpret_cast<uint64_t*>(p) = v;
    } else {
      for (uint32_t b = 0; b < n; ++b) p[b] = static_cast<uint8_t>(v >> (8 * b));
    }
  }
}

// fold_of_blob: the wrapped sum over samples of each sample's first
// min(8, bytes_per_sample) bytes read little-endian.
__global__ void fold_blob_kernel(const uint8_t* blob, uint64_t nsamples, uint32_t bps, unsigned long long* out) {
  unsigned long long acc = 0;
  const uint32_t n = bps < 8 ? bps : 8;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nsamples;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint8_t* p = blob + i * bps;
    uint64_t v = 0;
    for (uint32_t b = 0; b < n; ++b) v |= static_cast<uint64_t>(p[b]) << (8 * b);
    acc += v;
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

unsigned grid_for(uint64_t work_items, int threads) {
  const uint64_t want = (work_items + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(sm_count()) * 8;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min(want, cap)));
}

}  // namespace

cudaError_t launch_items(uint8_t* dst, const uint64_t* folds, uint32_t count, uint32_t sample_bytes,
                         cudaStream_t stream) {
  const uint64_t words = (sample_bytes + 7) / 8 * uint64_t(count);
  if (words == 0) return cudaSuccess;
  items_kernel<<<grid_for(words, 256), 256, 0, stream>>>(dst, folds, count, sample_bytes);
  return cudaGetLastError();
}

cudaError_t launch_fold_blob(const uint8_t* blob, uint64_t bytes, uint32_t bytes_per_sample,
                             unsigned long long* out, cudaStream_t stream) {
  const uint64_t ns = bytes_per_sample ? bytes / bytes_per_sample : 0;
  if (ns == 0) return cudaSuccess;
  fold_blob_kernel<<<grid_for(ns, 256), 256, 0, stream>>>(blob, ns, bytes_per_sample, out);
  return cudaGetLastError();
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

void retain_pool() {
  // The device's default stream-ordered pool returns memory to the driver at
  // every synchronize unless a release threshold is set; the synchronous
  // checkers (whole FNV scratch, blob check) would re-map it on every call.
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = 256ull << 20;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev] = true;
}

cudaError_t whole_fnv(const uint8_t* data, uint64_t len, uint64_t h0, uint64_t* out,
                      cudaStream_t stream) {
  retain_pool();
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
  const uint64_t offT = 0, offP = align_up(nsub * kSpecTab, 256), offLam = offP + align_up(nsub, 256),
                 offInit = offLam + align_up(nseg, 256), offF = offInit + align_up(nsub * 8, 256),
                 offOut = offF + align_up(nsub * 8, 256), total = offOut + 256;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), total, stream);
  if (e != cudaSuccess) return e;
  uint8_t* T = scratch + offT;
  uint8_t* P = scratch + offP;
  uint8_t* lam = scratch + offLam;
  uint64_t* init = reinterpret_cast<uint64_t*>(scratch + offInit);
  uint64_t* F = reinterpret_cast<uint64_t*>(scratch + offF);
  uint64_t* dout = reinterpret_cast<uint64_t*>(scratch + offOut);

  const uint64_t spec_threads = nseg * kSpecThreads;
  fnv_spec_kernel<<<static_cast<unsigned>((spec_threads + 255) / 256), 256, 0, stream>>>(
      data, len, Ls, nsub, T, P);
  fnv_walk_kernel<<<1, 512, 0, stream>>>(T, P, nsub, nseg, static_cast<uint32_t>(h0 & 0xff), lam);
  fnv_init_kernel<<<grid_for(nsub, 256), 256, 0, stream>>>(T, P, lam, nsub, init);
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
