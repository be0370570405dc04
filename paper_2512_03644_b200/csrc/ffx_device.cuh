// ffx_device.cuh -- device-side arithmetic shared by the ffx kernels.
//
// FNV-1a-64 (reference hash.cpp:102-110) and the splitmix64 finaliser
// (reference evolution.cpp:43-48), restated for 32-bit integer datapaths.
#pragma once

#include <cstdint>

namespace ffx {

constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ull;  // hash.cpp:104
constexpr uint64_t kFnvPrime = 0x100000001b3ull;       // hash.cpp:107 (= 2^40 + 0x1b3)
constexpr uint32_t kFnvQ = 0x1b3u;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;    // evolution.cpp:44, :76

// FNV-1a-64 state split in 32-bit halves.  With h = hi:lo and x = lo ^ b,
//   (h ^ b) * (2^40 + Q) mod 2^64  =  hi*Q*2^32 + x*2^40 + x*Q
// so lo' = lo32(x*Q) and hi' = hi*Q + hi32(x*Q) + (x << 8): one wide
// multiply, one multiply-add and one shift-add per byte.
// kAluShift selects how the (x << 8) add is issued -- see byte().
template <bool kAluShift>
struct FnvT {
  uint32_t lo, hi;

  __device__ __forceinline__ void init() {
    lo = static_cast<uint32_t>(kFnvBasis);
    hi = static_cast<uint32_t>(kFnvBasis >> 32);
  }
  __device__ __forceinline__ void set(uint64_t h) {
    lo = static_cast<uint32_t>(h);
    hi = static_cast<uint32_t>(h >> 32);
  }
  __device__ __forceinline__ uint64_t value() const {
    return (static_cast<uint64_t>(hi) << 32) | lo;
  }
  // Written as mul.lo/mul.hi/mad so ptxas folds hi32(x*Q) into the hi*Q
  // multiply-add (IMAD.WIDE + IMAD on the FMA-heavy pipe).  The (x << 8) add:
  //  * kAluShift = false: `t + (x << 8)`, which ptxas issues as IMAD x*256 + t
  //    for ~3/4 of the bytes (FMA-heavy) and LEA for the rest;
  //  * kAluShift = true: a funnel shift + add, which ptxas fuses into one
  //    LEA.HI on the ALU pipe, unloading the FMA-heavy pipe (66% busy in the
  //    fused kernel, ncu).
  // Same-box A/B (profiles/r1_fnv_alu_shift_ab_1gpu.txt): the ALU form makes
  // checksum-only launches 3.4% faster (3543-3551 -> 3666-3671 GB/s) but the
  // fused copy+hash kernel 0.7% slower (its ALU pipe also carries the TMA /
  // barrier bookkeeping), so the kernels pick per mode.  With no memory in
  // the way (tools/fnv_pipe_probe.cu) the ALU form is 5-25% faster.
  __device__ __forceinline__ void byte(uint32_t b) {
    const uint32_t x = lo ^ b;
    uint32_t plo, phi, t;
    asm("mul.lo.u32 %0, %2, 0x1b3;\n\tmul.hi.u32 %1, %2, 0x1b3;" : "=r"(plo), "=r"(phi) : "r"(x));
    asm("mad.lo.u32 %0, %1, 0x1b3, %2;" : "=r"(t) : "r"(hi), "r"(phi));
    if constexpr (kAluShift) {
      uint32_t s;
      asm("shf.l.wrap.b32 %0, %1, %2, 8;" : "=r"(s) : "r"(0u), "r"(x));  // x << 8
      asm("add.u32 %0, %1, %2;" : "=r"(hi) : "r"(t), "r"(s));
    } else {
      hi = t + (x << 8);
    }
    lo = plo;
  }
  // Four bytes of a little-endian word, in memory order.
  __device__ __forceinline__ void word(uint32_t w) {
    byte(w & 0xffu);
    byte(__byte_perm(w, 0u, 0x4441));
    byte(__byte_perm(w, 0u, 0x4442));
    byte(w >> 24);
  }
  __device__ __forceinline__ void vec(const uint4& v) {
    word(v.x);
    word(v.y);
    word(v.z);
    word(v.w);
  }
};
using Fnv = FnvT<false>;     // copy + hash kernels
using FnvAlu = FnvT<true>;   // checksum-only kernels

// evo::mix64 including its leading golden-ratio add (evolution.cpp:43-48).
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += kGolden;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Slot-metadata stores (SlotMeta words, SNP1 header, the COMMITTED flag).
// Through an NVSwitch multicast range (the double-neighbour target) they are
// multimem.st -- the only plain-store form the PTX ISA defines on a multimem
// address -- so every bound holder receives them; elsewhere volatile stores.
// Ordering is by the callers' system-scope fences, as before.
__device__ __forceinline__ void meta_st32(void* p, uint32_t v, bool mc) {
  if (mc) asm volatile("multimem.st.relaxed.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else *reinterpret_cast<volatile uint32_t*>(p) = v;
}
__device__ __forceinline__ void meta_st64(void* p, uint64_t v, bool mc) {
  if (mc) asm volatile("multimem.st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else *reinterpret_cast<volatile uint64_t*>(p) = v;
}
__device__ __forceinline__ void meta_st128(void* p, const uint4& v, bool mc) {
  meta_st64(p, (static_cast<uint64_t>(v.y) << 32) | v.x, mc);
  meta_st64(static_cast<uint8_t*>(p) + 8, (static_cast<uint64_t>(v.w) << 32) | v.z, mc);
}

// Streaming global accesses: every payload byte is touched once per pass.
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  return __ldcs(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  __stcs(reinterpret_cast<uint4*>(p), v);
}

}  // namespace ffx
