// Device helpers shared by the resident-factor persistent kernels (fold_res.cu: folded products,
// dense_res.cu: dense products): DMMA, 8-byte cp.async with zero fill, mbarrier ring primitives.
#pragma once

#include <cstdint>

namespace stiga {
namespace gpu {
namespace resdev {

__device__ __forceinline__ void rdmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned ru32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void rcp8(unsigned dst, const double* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void rmb_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(ru32(bar)), "r"(count));
}
__device__ __forceinline__ void rmb_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(ru32(bar)) : "memory");
}
// arrive on `bar` when every cp.async issued so far by this thread has landed (counts against the
// barrier's expected arrivals: .noinc)
__device__ __forceinline__ void rmb_cp_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(ru32(bar)) : "memory");
}
__device__ __forceinline__ void rmb_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "RWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra RWAIT_%=;\n"
        "}\n" ::"r"(ru32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ long long rbase(long long cc, long long L, int n) {
    if (L == 1) return cc * n;
    const long long r = cc / L;
    return (cc - r * L) + L * static_cast<long long>(n) * r;
}

}  // namespace resdev
}  // namespace gpu
}  // namespace stiga
