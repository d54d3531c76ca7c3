// stereo_common.cuh — device helpers and plan utilities shared by the
// kernel translation units of libstereo_b200.so (internal).
#pragma once
#include <cstdlib>

#include <algorithm>
#include "stereo_internal.cuh"

namespace stereo {

constexpr unsigned kFull = 0xffffffffu;
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// x pass geometry limits (stereo_xpass.cu; the planner sizes shared memory with them)
constexpr int kXMaxWarps = 16;
constexpr int kXMaxSlots = 4;
constexpr int kXFixExt = 128;  // compile-time prefix pitch extension (FIXPL)
constexpr int kXMaxC2 = 27;    // widest lane chunk kept in registers in one pass

// bulk copies and mbarriers (PTX idiom)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void xbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void xbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "XWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra XWAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Development knobs (plan overrides for tuning experiments; unset = the
// planner's choice).  Out-of-range values are clamped.
inline int env_int(const char* name, int dflt, int lo, int hi) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::max(lo, std::min(hi, std::atoi(v)));
}

// Kernels of different frames share SMs (frames in flight on several
// streams); an SM whose L1/shared carveout was sized for a small-shared-memory
// kernel cannot take an x-pass or y-pass CTA until it is reconfigured, so
// every kernel asks for the maximum shared carveout (STEREO_CARVEOUT = percent,
// -1 = the driver's default; measured identical on B200 today, where the
// driver already picks the maximum for these kernels: kept as a guarantee).
template <typename F>
inline cudaError_t max_carveout(F fn) {
  const int pct = env_int("STEREO_CARVEOUT", 100, -1, 100);
  if (pct < 0) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

// The dynamic shared-memory limit is a per-kernel, process-wide attribute:
// only ever RAISE it, so that a handle created later with a smaller footprint
// never breaks the launches of an earlier, larger one.
template <typename F>
inline cudaError_t raise_smem(F fn, int bytes) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  if (fa.maxDynamicSharedSizeBytes >= bytes) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}


cudaError_t setup_xpass(int C, int smem);  // shared-memory attributes of the x-pass kernels

}  // namespace stereo
