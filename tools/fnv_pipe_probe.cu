// FNV-1a-64 issue-cost probe: how many bytes/s can the SMs hash when memory is
// out of the picture?  Each lane loads 128 B once into registers and hashes
// them R times (one serial chain per lane, or two interleaved chains), at a
// chosen number of resident warps per SM.  Separates "latency-bound chain"
// (rate grows with warps / chains) from "pipe-bound" (rate flat).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fnv_pipe_probe tools/fnv_pipe_probe.cu
//   ./fnv_pipe_probe            -> one JSON line per (variant, warps/SM)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2512_03644_b200/csrc/ffx_device.cuh"

namespace {

using ffx::Fnv;

// B: the hi word as one IMAD + LEA feeding a 64-bit-addend IMAD.WIDE
struct FnvB {
  uint32_t lo, hi;
  __device__ __forceinline__ void byte(uint32_t b) {
    const uint32_t x = lo ^ b;
    const uint32_t t = hi * 0x1b3u + (x << 8);
    uint64_t r;
    asm("mad.wide.u32 %0, %1, 0x1b3, %2;" : "=l"(r) : "r"(x), "l"(static_cast<uint64_t>(t) << 32));
    lo = static_cast<uint32_t>(r);
    hi = static_cast<uint32_t>(r >> 32);
  }
  __device__ __forceinline__ void word(uint32_t w) {
    byte(w & 0xffu);
    byte(__byte_perm(w, 0u, 0x4441));
    byte(__byte_perm(w, 0u, 0x4442));
    byte(w >> 24);
  }
};

// D/E: the current mul.lo/mul.hi/mad, with (x << 8) moved off the FMA-heavy
// pipe: D builds it with PRMT (byte permute), E with a funnel shift; both add
// with IADD3 (ALU pipe) instead of the IMAD x*256 + t ptxas otherwise picks.
template <int How>
struct FnvD {
  uint32_t lo, hi;
  __device__ __forceinline__ void byte(uint32_t b) {
    const uint32_t x = lo ^ b;
    uint32_t plo, phi, t, s;
    asm("mul.lo.u32 %0, %2, 0x1b3;\n\tmul.hi.u32 %1, %2, 0x1b3;" : "=r"(plo), "=r"(phi) : "r"(x));
    asm("mad.lo.u32 %0, %1, 0x1b3, %2;" : "=r"(t) : "r"(hi), "r"(phi));
    if constexpr (How == 0) s = __byte_perm(x, 0u, 0x2104);
    else asm("shf.l.wrap.b32 %0, %1, %2, 8;" : "=r"(s) : "r"(0u), "r"(x));
    asm("add.u32 %0, %1, %2;" : "=r"(hi) : "r"(t), "r"(s));
    lo = plo;
  }
  __device__ __forceinline__ void word(uint32_t w) {
    byte(w & 0xffu);
    byte(__byte_perm(w, 0u, 0x4441));
    byte(__byte_perm(w, 0u, 0x4442));
    byte(w >> 24);
  }
};

// C: plain 64-bit C++ (what nvcc makes of h = (h ^ b) * P)
struct FnvC {
  uint64_t h;
  __device__ __forceinline__ void byte(uint32_t b) { h = (h ^ b) * 0x100000001b3ull; }
  __device__ __forceinline__ void word(uint32_t w) {
    byte(w & 0xffu);
    byte((w >> 8) & 0xffu);
    byte((w >> 16) & 0xffu);
    byte(w >> 24);
  }
};

template <int V, int CH>
__global__ void probe(const uint4* __restrict__ in, uint64_t* out, int reps) {
  const uint4* p = in + (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  uint4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = p[i];
  uint64_t acc = 0;
  if constexpr (V == 0) {
    Fnv h[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) h[c].set(0xcbf29ce484222325ull + c);
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) h[c].vec(v[(i + c) & 7]);
#pragma unroll
    for (int c = 0; c < CH; ++c) acc ^= h[c].value();
  } else if constexpr (V == 1) {
    FnvB h[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { h[c].lo = 0x84222325u + c; h[c].hi = 0xcbf29ce4u; }
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const uint4 w = v[(i + c) & 7];
          h[c].word(w.x); h[c].word(w.y); h[c].word(w.z); h[c].word(w.w);
        }
#pragma unroll
    for (int c = 0; c < CH; ++c) acc ^= (static_cast<uint64_t>(h[c].hi) << 32) | h[c].lo;
  } else if constexpr (V == 3 || V == 4) {
    FnvD<V - 3> h[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { h[c].lo = 0x84222325u + c; h[c].hi = 0xcbf29ce4u; }
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const uint4 w = v[(i + c) & 7];
          h[c].word(w.x); h[c].word(w.y); h[c].word(w.z); h[c].word(w.w);
        }
#pragma unroll
    for (int c = 0; c < CH; ++c) acc ^= (static_cast<uint64_t>(h[c].hi) << 32) | h[c].lo;
  } else {
    FnvC h[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) h[c].h = 0xcbf29ce484222325ull + c;
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const uint4 w = v[(i + c) & 7];
          h[c].word(w.x); h[c].word(w.y); h[c].word(w.z); h[c].word(w.w);
        }
#pragma unroll
    for (int c = 0; c < CH; ++c) acc ^= h[c].h;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V, int CH>
void run(const char* name, const uint4* in, uint64_t* out, int sms, int max_threads) {
  const int reps = 64;
  for (int warps_per_sm : {4, 8, 12, 16, 24, 32, 48}) {
    const int threads = 128;
    const int blocks_per_sm = warps_per_sm / 4;
    const int blocks = sms * blocks_per_sm;
    if (blocks * threads > max_threads) break;
    cudaFuncSetAttribute(probe<V, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
    // pin the residency: dynamic smem so that exactly blocks_per_sm fit per SM
    const int smem = (200 * 1024) / blocks_per_sm;
    cudaFuncSetAttribute(probe<V, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<V, CH><<<blocks, threads, smem>>>(in, out, 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<V, CH><<<blocks, threads, smem>>>(in, out, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = static_cast<double>(blocks) * threads * CH * 128.0 * reps;
    uint64_t h0 = 0;
    cudaMemcpy(&h0, out, 8, cudaMemcpyDeviceToHost);
    printf("{\"variant\": \"%s\", \"chains_per_lane\": %d, \"warps_per_sm\": %d, \"hash_gbs\": %.1f, "
           "\"lane0_hash\": \"%016llx\", \"err\": \"%s\"}\n",
           name, CH, warps_per_sm, bytes / (ms * 1e-3) / 1e9, static_cast<unsigned long long>(h0),
           cudaGetErrorString(cudaGetLastError()));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
}

}  // namespace

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int max_threads = sms * 48 * 32;
  uint4* in = nullptr;
  uint64_t* out = nullptr;
  cudaMalloc(&in, static_cast<size_t>(max_threads) * 128);
  cudaMalloc(&out, static_cast<size_t>(max_threads) * 8);
  cudaMemset(in, 0x5a, static_cast<size_t>(max_threads) * 128);
  run<0, 1>("Fnv::byte (ffx_device.cuh)", in, out, sms, max_threads);
  run<0, 2>("Fnv::byte (ffx_device.cuh)", in, out, sms, max_threads);
  run<1, 1>("wide-addend", in, out, sms, max_threads);
  run<1, 2>("wide-addend", in, out, sms, max_threads);
  run<3, 1>("shift-by-prmt", in, out, sms, max_threads);
  run<3, 2>("shift-by-prmt", in, out, sms, max_threads);
  run<4, 1>("shift-by-shf", in, out, sms, max_threads);
  run<4, 2>("shift-by-shf", in, out, sms, max_threads);
  run<2, 1>("plain-u64", in, out, sms, max_threads);
  run<2, 2>("plain-u64", in, out, sms, max_threads);
  return 0;
}
