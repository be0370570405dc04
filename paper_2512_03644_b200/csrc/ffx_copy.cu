// ffx_copy.cu -- copy-only TMA kernel and the stand-alone slot commit, for
// the slice scheduler's split policy.
//
// In a training step the snapshot competes with the step for two resources:
// NVLink (busy during the step's all-gathers / reduce-scatters) and SMs (busy
// during its GEMMs).  The fused kernel needs both at once.  The split policy
// pulls them apart:
//   * copy batches (this kernel) run in the compute gaps, when NVLink is
//     idle: one warp per CTA drives 1-D TMA bulk copies (32 KB per op,
//     S stages), so a handful of SMs saturate the link;
//   * hash batches (slice_kernel in Hash mode, reading the *local* state and
//     writing the checksum table into the peer slot) run in the
//     communication gaps, when SMs idle behind NCCL and HBM has headroom;
//   * the commit (commit_kernel) runs once both queues have drained.
// The state is immutable between the optimizer updates, so the copied bytes
// and the hashed bytes are the same bytes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "ffx_device.cuh"
#include "ffx_kernels.h"

namespace ffx {

namespace {

constexpr int kCopyChunk = 32 * 1024;
constexpr int kCopyStages = 4;
constexpr int kCopySmem = kCopyChunk * kCopyStages + 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "FFX_CWAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra FFX_CWAIT;\n\t}" ::"r"(bar),
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

// Chunk c of region r covers [c*kCopyChunk, min((c+1)*kCopyChunk, bytes)).
// Chunks of aligned regions move by TMA except a sub-16-byte remainder,
// which the warp copies bytewise; unaligned regions go bytewise entirely.
__global__ void __launch_bounds__(32) copy_kernel(const __grid_constant__ CopyJob job) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* buf = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bars[kCopyStages];
  const int lane = threadIdx.x;
  if (lane == 0) {  // WRITING before any payload byte
    for (const SlotMark* mk : {&job.mark, &job.mark2}) {
      if (mk->slot == nullptr) continue;
      SlotMeta* m = reinterpret_cast<SlotMeta*>(mk->slot);
      const bool mc = mk->mcast != 0;
      meta_st32(&m->magic, kSlotMagic, mc);
      meta_st64(&m->iteration, mk->iteration, mc);
      meta_st64(&m->seq, mk->seq, mc);
      meta_st32(&m->state, kSlotWriting, mc);
    }
    __threadfence_system();
  }
  if (lane == 0) {
    for (int s = 0; s < kCopyStages; ++s) mbar_init(smem_u32(&bars[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;
  int inflight = 0;  // stages holding a load or an unfinished store read
  // Static round-robin over this launch's chunks, kCopyStages deep.
  const uint64_t lo = job.chunk_lo + blockIdx.x, hi = job.chunk_hi, step = gridDim.x;
  auto region_of = [&](uint64_t c) {
    int r = 0;
#pragma unroll
    for (int i = 1; i < static_cast<int>(kMaxRegions); ++i)
      if (i < static_cast<int>(job.nregions) && c >= job.chunk_base[i]) r = i;
    return r;
  };
  // Pass 1 (lane 0): TMA for the 16-byte-aligned part of every chunk.
  if (lane == 0) {
    uint64_t issue = lo;
    int slot_issue = 0, slot_done = 0;
    uint64_t done = lo;
    auto issue_one = [&](uint64_t c, int s) -> bool {
      const int r = region_of(c);
      const CopyRegion& R = job.reg[r];
      if (!R.aligned) return false;
      const uint64_t off = (c - job.chunk_base[r]) * kCopyChunk;
      const uint64_t len = (R.bytes - off < kCopyChunk ? R.bytes - off : kCopyChunk) & ~uint64_t{15};
      if (len == 0) return false;
      const uint32_t b = smem_u32(&bars[s]);
      mbar_expect_tx(b, static_cast<uint32_t>(len));
      bulk_load(smem_u32(buf + s * kCopyChunk), R.src + off, static_cast<uint32_t>(len), b);
      return true;
    };
    bool pending[kCopyStages] = {};
    uint64_t which[kCopyStages] = {};
    for (; issue < hi && inflight < kCopyStages; issue += step, ++inflight) {
      pending[slot_issue] = issue_one(issue, slot_issue);
      which[slot_issue] = issue;
      slot_issue = (slot_issue + 1) % kCopyStages;
    }
    while (done < hi) {
      const int s = slot_done;
      if (pending[s]) {
        mbar_wait(smem_u32(&bars[s]), (phase >> s) & 1u);
        const uint64_t c = which[s];
        const int r = region_of(c);
        const CopyRegion& R = job.reg[r];
        const uint64_t off = (c - job.chunk_base[r]) * kCopyChunk;
        const uint64_t len = (R.bytes - off < kCopyChunk ? R.bytes - off : kCopyChunk) & ~uint64_t{15};
        bulk_store(R.dst + off, smem_u32(buf + s * kCopyChunk), static_cast<uint32_t>(len));
        if (R.dst2 != nullptr)  // double neighbour: one load, two stores
          bulk_store(R.dst2 + off, smem_u32(buf + s * kCopyChunk), static_cast<uint32_t>(len));
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      phase ^= pending[s] ? (1u << s) : 0u;
      done += step;
      slot_done = (slot_done + 1) % kCopyStages;
      if (issue < hi) {
        // refill stage s once its store has finished reading shared memory
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        pending[s] = issue_one(issue, s);
        which[s] = issue;
        issue += step;
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncwarp();
  // Pass 2 (whole warp): remainders of aligned chunks and unaligned regions.
  for (uint64_t c = lo; c < hi; c += step) {
    const int r = region_of(c);
    const CopyRegion& R = job.reg[r];
    const uint64_t off = (c - job.chunk_base[r]) * kCopyChunk;
    const uint64_t end = R.bytes - off < kCopyChunk ? R.bytes : off + kCopyChunk;
    const uint64_t from = R.aligned ? off + ((end - off) & ~uint64_t{15}) : off;
    for (uint64_t o = from + lane; o < end; o += 32) {
      R.dst[o] = R.src[o];
      if (R.dst2 != nullptr) R.dst2[o] = R.src[o];
    }
  }
}

#ifdef FFX_DEV
// SM copy (measurement reference for the probe, FFX_COPY_SM=1): grid-stride
// 16-byte loads / stores, 4 in flight per thread.
__global__ void __launch_bounds__(256) sm_copy_kernel(const __grid_constant__ CopyJob job) {
  for (uint32_t r = 0; r < job.nregions; ++r) {
    const CopyRegion& R = job.reg[r];
    const uint64_t nv = R.bytes / 16;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint4* s = reinterpret_cast<const uint4*>(R.src);
    uint4* d = reinterpret_cast<uint4*>(R.dst);
    uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < nv; i += 4 * stride) {
      const uint4 a = ld_stream(s + i), b = ld_stream(s + i + stride), c = ld_stream(s + i + 2 * stride),
                  e = ld_stream(s + i + 3 * stride);
      st_stream(d + i, a);
      st_stream(d + i + stride, b);
      st_stream(d + i + 2 * stride, c);
      st_stream(d + i + 3 * stride, e);
    }
    for (; i < nv; i += stride) st_stream(d + i, ld_stream(s + i));
    if (blockIdx.x == 0 && threadIdx.x < R.bytes % 16) R.dst[nv * 16 + threadIdx.x] = R.src[nv * 16 + threadIdx.x];
  }
}
#endif  // FFX_DEV

// Single thread: the final slot commit (meta, SNP1 header, then COMMITTED).
__global__ void commit_kernel(const __grid_constant__ SlotCommit c) {
  __threadfence_system();
  const bool mc = c.mcast != 0;
  for (int i = 1; i < static_cast<int>(kMetaBytes / 16); ++i) meta_st128(c.slot + 16 * i, c.meta[i], mc);
  for (int i = 0; i < 2; ++i) meta_st128(c.slot + c.payload_off - 32 + 16 * i, c.snp1[i], mc);
  __threadfence_system();
  meta_st32(&reinterpret_cast<SlotMeta*>(c.slot)->state, kSlotCommitted, mc);
  __threadfence_system();
  if (c.ack != nullptr) {
    *reinterpret_cast<volatile uint64_t*>(c.ack) = c.ack_value;
    __threadfence_system();
  }
}

}  // namespace

void finalize_copy_job(CopyJob& job) {
  uint64_t chunks = 0;
  for (uint32_t r = 0; r < job.nregions; ++r) {
    job.chunk_base[r] = chunks;
    job.reg[r].aligned = (reinterpret_cast<uintptr_t>(job.reg[r].src) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(job.reg[r].dst) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(job.reg[r].dst2) % 16 == 0);
    chunks += (job.reg[r].bytes + kCopyChunk - 1) / kCopyChunk;
  }
  for (uint32_t r = job.nregions; r < kMaxRegions; ++r) job.chunk_base[r] = ~0ull;
  job.total_chunks = chunks;
  job.chunk_lo = 0;
  job.chunk_hi = chunks;
}

cudaError_t launch_copy(const CopyJob& job, uint32_t ctas, cudaStream_t stream) {
  static uint64_t set_on = 0;  // bit d: the shared-memory opt-in done on device d
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(set_on & bit)) {
    cudaError_t e = cudaFuncSetAttribute(copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kCopySmem);
    if (e != cudaSuccess) return e;
    set_on |= bit;
  }
#ifdef FFX_DEV
  static const bool sm = std::getenv("FFX_COPY_SM") != nullptr;
  if (sm && job.chunk_lo == 0 && job.chunk_hi == job.total_chunks && job.mark.slot == nullptr) {
    sm_copy_kernel<<<ctas ? ctas : 148 * 8, 256, 0, stream>>>(job);
    return cudaGetLastError();
  }
#endif
  const uint64_t n = job.chunk_hi - job.chunk_lo;
  const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(n, ctas ? ctas : 16));
  copy_kernel<<<static_cast<unsigned>(grid), 32, kCopySmem, stream>>>(job);
  return cudaGetLastError();
}

cudaError_t launch_mark(const SlotCommit& c, const SlotCommit* c2, cudaStream_t stream) {
  CopyJob mark{};
  mark.mark = SlotMark{c.slot, c.iteration, c.seq, c.mcast, 0};
  if (c2) mark.mark2 = SlotMark{c2->slot, c2->iteration, c2->seq, c2->mcast, 0};
  finalize_copy_job(mark);
  mark.chunk_lo = mark.chunk_hi = 0;
  return launch_copy(mark, 1, stream);
}

cudaError_t launch_commit(const SlotCommit& c, cudaStream_t stream) {
  commit_kernel<<<1, 1, 0, stream>>>(c);
  return cudaGetLastError();
}

}  // namespace ffx
