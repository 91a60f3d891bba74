// Cross-SM communication primitives shared by the persistent engines
// (engine.cu, engine2.cu): self-validating tagged 64-bit words (round tag in
// the top 16 bits, payload below), relaxed / acquire / release accesses at GPU
// scope, async proposal copies and the phase timers.
#pragma once
#include <cstdint>

namespace gcmcb {

constexpr uint64_t kPay = 0xffffffffffffull;

__device__ __forceinline__ uint64_t tagw(uint32_t r, uint64_t payload) {
  return ((uint64_t)(r & 0xffffu) << 48) | (payload & kPay);
}
__device__ __forceinline__ bool tagged(uint64_t w, uint32_t r) {
  return (uint32_t)(w >> 48) == (r & 0xffffu);
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void nap() { __nanosleep(20); }
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Phase timers: accumulated clock64 cycles per phase. Compiled in only with
// -DGCMC_PHASE_TIMERS (tools/build_variant.py prof -DGCMC_PHASE_TIMERS, then
// GCMC_LIB=... GCMC_ENGINE_PROFILE=1): twelve live 64-bit counters in every
// thread of the persistent kernel cost registers (and spills) otherwise.
#ifdef GCMC_PHASE_TIMERS
struct PhaseClock {
  unsigned long long acc[12] = {0};
  unsigned long long t = 0;
  bool on = false;
  __device__ __forceinline__ void start(bool enable) {
    on = enable;
    if (on) t = clock64();
  }
  __device__ __forceinline__ void mark(int k) {
    if (!on) return;
    const unsigned long long n = clock64();
    acc[k] += n - t;
    t = n;
  }
  __device__ __forceinline__ void flush(unsigned long long* p) {
    if (!on) return;
    for (int k = 0; k < 12; ++k) p[k] = acc[k];
  }
};
#else
struct PhaseClock {
  static constexpr bool on = false;
  unsigned long long acc[12];
  __device__ __forceinline__ void start(bool) {}
  __device__ __forceinline__ void mark(int) {}
  __device__ __forceinline__ void flush(unsigned long long*) {}
};
#endif

}  // namespace gcmcb
