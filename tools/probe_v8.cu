// probe_v8.cu -- does the store width of SM-issued peer writes move the
// NVLink ceiling?  (measurement tooling, not product code)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_v8 tools/probe_v8.cu
//   tools/probe_v8 [bytes]
//
// Two GPUs, both directions at once (the 2-rank ring shift): each GPU copies
// `bytes` from its own HBM into a buffer on the other GPU with
//   st128  plain 128-bit ld/st per thread (LDG/STG.128)
//   st256  Blackwell 256-bit ld/st (LDG/STG.E.ENL2.256)
//   ce     cudaMemcpyPeerAsync (copy engines)
// and, for reference, the same kernels pulling (peer loads, local stores).
// Prints one JSON line of per-GPU GB/s (best of 5 after warm-up).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                               \
    }                                                                             \
  } while (0)

__global__ void copy128(uint4* __restrict__ d, const uint4* __restrict__ s, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

__global__ void copy256(float* __restrict__ d, const float* __restrict__ s, size_t n32) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n32; i += (size_t)gridDim.x * blockDim.x) {
    float a0, a1, a2, a3, a4, a5, a6, a7;
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(a4), "=f"(a5), "=f"(a6), "=f"(a7)
                 : "l"(s + 8 * i));
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(d + 8 * i), "f"(a0), "f"(a1), "f"(a2),
                 "f"(a3), "f"(a4), "f"(a5), "f"(a6), "f"(a7)
                 : "memory");
  }
}

int main(int argc, char** argv) {
  const size_t bytes = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : (size_t(2336416800) / 32 * 32);
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    std::printf("{\"skipped\": \"needs 2 GPUs\"}\n");
    return 0;
  }
  void *src[2], *dst[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMalloc(&dst[g], bytes));
    CK(cudaMemset(src[g], 0x11 * (g + 1), bytes));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  // mode: 0 st128 push, 1 st256 push, 2 ce push, 3 st128 pull, 4 st256 pull
  auto run = [&](int mode, int g, int ctas_per_sm) {
    const int p = 1 - g;
    const bool pull = mode >= 3;
    void* d = pull ? dst[g] : dst[p];  // push: write the peer; pull: read the peer
    const void* s = pull ? src[p] : src[g];
    const int grid = sms * ctas_per_sm;
    if (mode == 0 || mode == 3)
      copy128<<<grid, 512, 0, st[g]>>>(static_cast<uint4*>(d), static_cast<const uint4*>(s), bytes / 16);
    else if (mode == 1 || mode == 4)
      copy256<<<grid, 512, 0, st[g]>>>(static_cast<float*>(d), static_cast<const float*>(s), bytes / 32);
    else
      CK(cudaMemcpyPeerAsync(d, p, s, g, bytes, st[g]));
  };
  const char* names[] = {"st128_push", "st256_push", "ce_push", "st128_pull", "st256_pull"};
  std::printf("{\"bytes\": %zu", bytes);
  for (int mode = 0; mode < 5; ++mode)
    for (int cps : {1, 2, 4}) {
      if (mode == 2 && cps > 1) continue;
      double best = 0;
      for (int rep = 0; rep < 6; ++rep) {
        for (int g = 0; g < 2; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaDeviceSynchronize());
        }
        for (int g = 0; g < 2; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventRecord(e0[g], st[g]));
          run(mode, g, cps);
          CK(cudaEventRecord(e1[g], st[g]));
        }
        float ms = 0;
        for (int g = 0; g < 2; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventSynchronize(e1[g]));
          float m = 0;
          CK(cudaEventElapsedTime(&m, e0[g], e1[g]));
          if (m > ms) ms = m;
        }
        if (rep > 0 && bytes / (ms * 1e-3) / 1e9 > best) best = bytes / (ms * 1e-3) / 1e9;
      }
      if (mode == 2) std::printf(", \"%s\": %.1f", names[mode], best);
      else std::printf(", \"%s_%dcta\": %.1f", names[mode], cps, best);
    }
  std::printf("}\n");
  return 0;
}
