// lb_tma.cuh -- asynchronous-copy building blocks for the step kernels (sm_90+ PTX):
// mbarriers, TMA tensor copies with L2 cache hints, cp.async, gpu-scope relaxed
// accesses, plus the host-side tensor-map encoder.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "lb_kernels.cuh"

namespace lbk {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// TMA 3-D tile copy global -> this CTA's shared memory, completing on `bar`.
// The box start must be 16-byte aligned in x (even fp64 index).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// L2 policies
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// kind: 0 evict_normal, 1 evict_first, 2 evict_last, 3 evict_unchanged
template <int KIND>
__device__ __forceinline__ unsigned long long policy_of() {
  unsigned long long p;
  if constexpr (KIND == 0) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  else if constexpr (KIND == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else if constexpr (KIND == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long policy_rt(int kind) {
  return kind == 0 ? policy_of<0>() : (kind == 1 ? policy_of<1>() : (kind == 2 ? policy_of<2>() : policy_of<3>()));
}
// store with an L2 policy
__device__ __forceinline__ void st_hint(double* a, double v, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// per-thread async copies (16 B needs 16-byte aligned source and destination)
template <int VEC>
__device__ __forceinline__ void cp_async_v(void* dst, const double* src) {
  if constexpr (VEC == 2)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The phi exchange between CTAs of one launch: relaxed gpu-scope (strong) loads and
// stores, so a value one CTA publishes and another reads is not a data race under
// the PTX memory model (an aligned 64-bit strong access is single-copy atomic: the
// reader sees the old or the new value, never a mix).  No ordering is needed --
// the value is its own flag (kXchEmpty).
__device__ __forceinline__ double ld_relaxed_f64(const double* a) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* a, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(a), "d"(v) : "memory");
}

// f / g components in slot order (d3q19.cuh): three contiguous runs each
//   f: 0..4 | 10..18 | 28..32      g: 5..9 | 19..27 | 33..37
__host__ __device__ constexpr int fslot_of_rank(int j) { return j < 5 ? j : (j < 14 ? 10 + (j - 5) : 28 + (j - 14)); }
__host__ __device__ constexpr int gslot_of_rank(int j) { return j < 5 ? 5 + j : (j < 14 ? 19 + (j - 5) : 33 + (j - 14)); }
__host__ __device__ constexpr int frank(int i) {  // canonical i -> rank
  return slot(0, i) < 5 ? slot(0, i) : (slot(0, i) < 19 ? slot(0, i) - 10 + 5 : slot(0, i) - 28 + 14);
}
__host__ __device__ constexpr int grank(int i) {
  return slot(1, i) < 10 ? slot(1, i) - 5 : (slot(1, i) < 28 ? slot(1, i) - 19 + 5 : slot(1, i) - 33 + 14);
}
// first slot of run r (0, 1, 2) of f (dist 0) or g (dist 1), and its length
__host__ __device__ constexpr int run_first(int dist, int r) { return (r == 0 ? 0 : (r == 1 ? 10 : 28)) + (dist ? (r == 1 ? 9 : 5) : 0); }
__host__ __device__ constexpr int run_len(int r) { return r == 1 ? 9 : 5; }
__host__ __device__ constexpr int run_rank0(int r) { return r == 0 ? 0 : (r == 1 ? 5 : 14); }

// host: 3-D fp64 tensor map of a distribution buffer {x: nx, y: ny, comp-plane: (nzl+2GZ)*38}
bool encode_dist_map(CUtensorMap* m, const Geom& G, const double* buf, unsigned bx, unsigned by, unsigned bz);
// host: 3-D fp64 tensor map of a phi buffer {x: nx, y: ny, plane: nzl+2GP}, boxes bx x by x 1
bool encode_phi_map(CUtensorMap* m, const Geom& G, const double* phi, unsigned bx, unsigned by);

}  // namespace lbk
