// mc_probe.cu -- standalone probe: can the snapshot kernel replicate into the
// dp+1 and dp+2 replica slots with ONE NVLink egress (NVSwitch multicast,
// SURVEY 8(f)-2) instead of two unicast stores?
//
// Single process, all visible GPUs.  Builds a multicast object over GPUs
// {0 (origin), 1, 2 (if present)}, binds a VMM allocation on each, maps the
// multicast range on GPU 0 and measures, for the same bytes:
//   unicast  : st.global.v4 into GPU 1's memory over P2P (today's path)
//   mm_st    : multimem.st.v4 into the multicast range (every member receives it)
//   st_mc    : a plain st.global.v4 to the multicast range
//   tma_mc   : cp.async.bulk (shared -> global) to the multicast range
// and checks bit-exactly what landed in every member's memory.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//            -o tools/mc_probe tools/mc_probe.cu -lcuda  Groups:
// {0,1}; {0,1,2}; {0,1,2} with the origin binding no memory; shareable-handle
// round trips (POSIX fd, fabric).  Prints one JSON line per group.  Not part
// of libffx.so.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    CUresult r_ = (x);                                                                \
    if (r_ != CUDA_SUCCESS) {                                                         \
      const char* s_ = nullptr;                                                       \
      cuGetErrorString(r_, &s_);                                                      \
      std::printf("{\"error\": \"%s -> %s (line %d)\"}\n", #x, s_ ? s_ : "?", __LINE__); \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)
#define RK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::printf("{\"error\": \"%s -> %s (line %d)\"}\n", #x, cudaGetErrorString(e_), __LINE__); \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ uint4 pattern(uint64_t i, uint32_t seed) {
  uint64_t z = i * 0x9E3779B97F4A7C15ull + seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return make_uint4(static_cast<uint32_t>(z), static_cast<uint32_t>(z >> 32), static_cast<uint32_t>(~z),
                    static_cast<uint32_t>(z >> 17));
}

__global__ void k_st(uint4* dst, uint64_t n16, uint32_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = pattern(i, seed);
}

__global__ void k_mm_st(uint4* mc, uint64_t n16, uint32_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = pattern(i, seed);
    asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  }
}

// One warp per CTA: stage a 16 KB chunk of `src` in shared memory (bulk load),
// then bulk-store it to `dst` (the multicast range).
__global__ void k_tma(const uint8_t* src, uint8_t* dst, uint64_t bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  constexpr uint32_t kChunk = 16384;
  const uint32_t sbar = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  const uint32_t sdat = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t phase = 0;
  for (uint64_t o = blockIdx.x * (uint64_t)kChunk; o < bytes; o += (uint64_t)gridDim.x * kChunk) {
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(kChunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sdat),
                   "l"(src + o), "r"(kChunk), "r"(sbar)
                   : "memory");
      asm volatile(
          "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(sbar),
          "r"(phase));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + o), "r"(sdat), "r"(kChunk)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;");
    }
    phase ^= 1;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_cmp(const uint4* got, uint64_t n16, uint32_t seed, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 a = got[i], b = pattern(i, seed);
    if (a.x != b.x || a.y != b.y || a.z != b.z || a.w != b.w) atomicAdd(bad, 1ull);
  }
}


struct Member {
  int dev;
  bool bound;
  CUmemGenericAllocationHandle h;
  CUdeviceptr va;  // unicast mapping, accessible from the member and GPU 0
};

static int g_sms = 0;
static uint8_t* g_src = nullptr;
static unsigned long long* g_bad = nullptr;

#define CKR(x)                                                                        \
  do {                                                                                \
    CUresult r_ = (x);                                                                \
    if (r_ != CUDA_SUCCESS) {                                                         \
      const char* s_ = nullptr;                                                       \
      cuGetErrorString(r_, &s_);                                                      \
      out += std::string(", \"error\": \"") + #x + " -> " + (s_ ? s_ : "?") + "\"";   \
      return out + "}";                                                               \
    }                                                                                 \
  } while (0)
#define RKR(x)                                                                        \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      out += std::string(", \"error\": \"") + #x + " -> " + cudaGetErrorString(e_) + "\""; \
      return out + "}";                                                               \
    }                                                                                 \
  } while (0)

// One multicast team: GPUs devs[0..k) (devs[0] writes), bind[i] = member i binds
// memory; alias_sink: the writer binds ONE minimum-granularity chunk at every
// offset of the range instead (a sink that costs 2 MB, not the replica size).
static std::string run_group(const char* name, std::vector<int> devs, std::vector<bool> bind, uint64_t bytes,
                             CUmemAllocationHandleType ht, bool alias_sink = false, bool writer_member = true) {
  std::string out = std::string("{\"group\": \"") + name + "\", \"devs\": [";
  for (size_t i = 0; i < devs.size(); ++i) out += (i ? "," : "") + std::to_string(devs[i]);
  out += "]";
  const int k = static_cast<int>(devs.size());
  CUmulticastObjectProp prop{};
  prop.numDevices = writer_member ? k : k - 1;
  prop.handleTypes = ht;
  prop.size = bytes;
  size_t gmin = 0, grec = 0;
  CKR(cuMulticastGetGranularity(&gmin, &prop, CU_MULTICAST_GRANULARITY_MINIMUM));
  CKR(cuMulticastGetGranularity(&grec, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  out += ", \"gran_min\": " + std::to_string(gmin) + ", \"gran_rec\": " + std::to_string(grec);
  const uint64_t size = (bytes + grec - 1) / grec * grec;
  prop.size = size;
  CUmemGenericAllocationHandle mch;
  CKR(cuMulticastCreate(&mch, &prop));
  if (ht == CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) {  // shareable round trip through an fd
    int fd = -1;
    CKR(cuMemExportToShareableHandle(&fd, mch, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    CUmemGenericAllocationHandle imp;
    CKR(cuMemImportFromShareableHandle(&imp, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                                       CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    out += ", \"fd_roundtrip\": true";
    cuMemRelease(imp);
  } else if (ht == CU_MEM_HANDLE_TYPE_FABRIC) {
    CUmemFabricHandle fh;
    CKR(cuMemExportToShareableHandle(&fh, mch, CU_MEM_HANDLE_TYPE_FABRIC, 0));
    CUmemGenericAllocationHandle imp;
    CKR(cuMemImportFromShareableHandle(&imp, &fh, CU_MEM_HANDLE_TYPE_FABRIC));
    out += ", \"fabric_roundtrip\": true";
    cuMemRelease(imp);
  }
  for (int i = writer_member ? 0 : 1; i < k; ++i) {
    CUdevice d;
    CKR(cuDeviceGet(&d, devs[i]));
    CKR(cuMulticastAddDevice(mch, d));
  }
  std::vector<Member> m(k);
  for (int i = 0; i < k; ++i) {
    m[i].dev = devs[i];
    m[i].bound = bind[i];
    m[i].va = 0;
    if (i == 0 && alias_sink) {
      CUmemAllocationProp ap{};
      ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
      ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ap.location.id = devs[0];
      ap.requestedHandleTypes = ht;
      CKR(cuMemCreate(&m[0].h, gmin, &ap, 0));
      for (uint64_t o = 0; o < size; o += gmin) CKR(cuMulticastBindMem(mch, o, m[0].h, 0, gmin, 0));
      out += ", \"alias_sink_binds\": " + std::to_string(size / gmin);
      continue;
    }
    if (!bind[i]) continue;
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = devs[i];
    ap.requestedHandleTypes = ht;
    CKR(cuMemCreate(&m[i].h, size, &ap, 0));
    CKR(cuMulticastBindMem(mch, 0, m[i].h, 0, size, 0));
    CKR(cuMemAddressReserve(&m[i].va, size, grec, 0, 0));
    CKR(cuMemMap(m[i].va, size, 0, m[i].h, 0));
    CUmemAccessDesc acc[2] = {};
    acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[0].location.id = devs[i];
    acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    acc[1] = acc[0];
    acc[1].location.id = devs[0];
    CKR(cuMemSetAccess(m[i].va, size, acc, devs[i] == devs[0] ? 1 : 2));
  }
  CUdeviceptr mcva;
  CKR(cuMemAddressReserve(&mcva, size, grec, 0, 0));
  CKR(cuMemMap(mcva, size, 0, mch, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = devs[0];
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CKR(cuMemSetAccess(mcva, size, &acc, 1));

  const uint64_t n16 = bytes / 16;
  cudaEvent_t e0, e1;
  RKR(cudaSetDevice(devs[0]));
  RKR(cudaEventCreate(&e0));
  RKR(cudaEventCreate(&e1));
  auto clear = [&]() -> cudaError_t {
    for (int i = 0; i < k; ++i) {
      if (!m[i].bound) continue;
      cudaSetDevice(m[i].dev);
      cudaMemset(reinterpret_cast<void*>(m[i].va), 0, bytes);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) return e;
    }
    return cudaSetDevice(devs[0]);
  };
  auto check = [&](uint32_t seed) -> std::string {
    std::string c = "[";
    for (int i = 0; i < k; ++i) {
      if (!m[i].bound) {
        c += std::string(i ? "," : "") + "null";
        continue;
      }
      cudaSetDevice(m[i].dev);
      g_bad[0] = 0;
      k_cmp<<<g_sms * 4, 256>>>(reinterpret_cast<const uint4*>(m[i].va), n16, seed, g_bad);
      cudaDeviceSynchronize();
      c += (i ? "," : "") + std::to_string(g_bad[0]);
    }
    cudaSetDevice(devs[0]);
    return c + "]";
  };
  auto timed = [&](auto launch) -> double {
    for (int w = 0; w < 2; ++w) launch();
    cudaDeviceSynchronize();
    const int reps = 5;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return bytes * (double)reps / (ms / 1e3) / 1e9;
  };
  const unsigned grid = g_sms * 8;
  RKR(clear());
  double g = timed([&] { k_mm_st<<<grid, 256>>>(reinterpret_cast<uint4*>(mcva), n16, 22); });
  RKR(cudaGetLastError());
  out += ", \"multimem_st_gbs\": " + std::to_string(g) + ", \"multimem_bad\": " + check(22);
  RKR(clear());
  g = timed([&] { k_tma<<<g_sms * 4, 32, 16384>>>(g_src, reinterpret_cast<uint8_t*>(mcva), bytes); });
  RKR(cudaGetLastError());
  out += ", \"tma_bulk_to_mc_gbs\": " + std::to_string(g) + ", \"tma_bad\": " + check(44);
  // unicast references from the same writer into member 1
  if (k > 1 && m[1].bound) {
    RKR(clear());
    g = timed([&] { k_tma<<<g_sms * 4, 32, 16384>>>(g_src, reinterpret_cast<uint8_t*>(m[1].va), bytes); });
    out += ", \"tma_unicast_peer_gbs\": " + std::to_string(g);
    if (k > 2 && m[2].bound) {  // today's double-neighbour: two unicast stores of every tile
      RKR(clear());
      g = timed([&] {
        k_tma<<<g_sms * 2, 32, 16384>>>(g_src, reinterpret_cast<uint8_t*>(m[1].va), bytes);
        k_tma<<<g_sms * 2, 32, 16384>>>(g_src, reinterpret_cast<uint8_t*>(m[2].va), bytes);
      });
      out += ", \"tma_two_unicast_serial_gbs_per_copy\": " + std::to_string(g);
    }
  }
  cudaDeviceSynchronize();
  cuMemUnmap(mcva, size);
  cuMemAddressFree(mcva, size);
  for (int i = 0; i < k; ++i) {
    if (!m[i].bound) continue;
    CUdevice d;
    cuDeviceGet(&d, m[i].dev);
    cuMulticastUnbind(mch, d, 0, size);
    cuMemUnmap(m[i].va, size);
    cuMemAddressFree(m[i].va, size);
    cuMemRelease(m[i].h);
  }
  cuMemRelease(mch);
  return out + "}";
}

int main(int argc, char** argv) {
  const uint64_t bytes = (argc > 1 ? std::strtoull(argv[1], nullptr, 0) : (1ull << 30));
  CK(cuInit(0));
  int n = 0;
  CK(cuDeviceGetCount(&n));
  std::string attrs = "{\"gpus\": " + std::to_string(n) + ", \"attrs\": [";
  for (int d = 0; d < n; ++d) {
    CUdevice dev;
    CK(cuDeviceGet(&dev, d));
    int mc = 0, fab = 0, fd = 0;
    CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    CK(cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev));
    CK(cuDeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev));
    attrs += std::string(d ? "," : "") + "{\"multicast\": " + std::to_string(mc) + ", \"fabric\": " +
             std::to_string(fab) + ", \"posix_fd\": " + std::to_string(fd) + "}";
  }
  std::printf("%s]}\n", attrs.c_str());
  std::fflush(stdout);
  if (n < 2) return 0;
  for (int i = 0; i < n; ++i) {
    RK(cudaSetDevice(i));
    for (int j = 0; j < n; ++j)
      if (j != i) cudaDeviceEnablePeerAccess(j, 0);
  }
  cudaGetLastError();
  RK(cudaSetDevice(0));
  RK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
  RK(cudaMalloc(&g_src, bytes));
  RK(cudaMallocManaged(&g_bad, 64));
  k_st<<<g_sms * 8, 256>>>(reinterpret_cast<uint4*>(g_src), bytes / 16, 44);
  RK(cudaDeviceSynchronize());
  RK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  const auto FD = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  std::printf("%s\n", run_group("origin+1", {0, 1}, {true, true}, bytes, FD).c_str());
  std::fflush(stdout);
  if (n >= 3) {
    std::printf("%s\n", run_group("origin+2", {0, 1, 2}, {true, true, true}, bytes, FD).c_str());
    std::fflush(stdout);
  }
  if (n >= 3) {
    std::printf("%s\n",
                run_group("writer_outside_team", {0, 1, 2}, {false, true, true}, bytes, FD, false, false).c_str());
    std::fflush(stdout);
    std::printf("%s\n", run_group("origin_alias_sink+2", {0, 1, 2}, {false, true, true}, bytes, FD, true).c_str());
    std::fflush(stdout);
    std::printf("%s\n", run_group("2_holders_only", {0, 1, 2}, {false, true, true}, bytes, FD).c_str());
    std::fflush(stdout);
  }
  return 0;
}
