// ptx.cuh — thin inline-PTX wrappers for sm_100a used by the SySTeC kernels:
// mbarrier + 1-D bulk async copy (TMA engine, SASS UBLKCP), L2 cache-policy
// hints, and vector reductions into global memory (SASS REDG.E.ADD.F32x4).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace systec {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier --------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- L2 cache policies -----------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ---- 1-D bulk copy global -> shared (completes on an mbarrier) -------------
// dst, src and bytes must be multiples of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// ---- gathers ------------------------------------------------------------------
#ifdef SYSTEC_L1_NOALLOC
#define SYSTEC_LD_L1 ".L1::no_allocate"
#else
#define SYSTEC_LD_L1 ""
#endif
__device__ __forceinline__ float4 ldg4_hint(const float *p, uint64_t policy) {
    float4 v;
    asm volatile("ld.global.nc" SYSTEC_LD_L1 ".L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(policy));
    return v;
}
// 8 floats, one 32-byte load (sm_100a LDG.E.ENL2.256); p 32-byte aligned
struct float8 {
    float4 lo, hi;
};
__device__ __forceinline__ float8 ldg8_hint(const float *p, uint64_t policy) {
    float8 v;
    asm volatile("ld.global.nc" SYSTEC_LD_L1 ".L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=f"(v.lo.x), "=f"(v.lo.y), "=f"(v.lo.z), "=f"(v.lo.w), "=f"(v.hi.x), "=f"(v.hi.y),
                   "=f"(v.hi.z), "=f"(v.hi.w)
                 : "l"(p), "l"(policy));
    return v;
}
__device__ __forceinline__ float ldg1_hint(const float *p, uint64_t policy) {
    float v;
    asm volatile("ld.global.nc" SYSTEC_LD_L1 ".L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(policy));
    return v;
}
__device__ __forceinline__ float4 ldg4(const float *p) {
    return __ldg(reinterpret_cast<const float4 *>(p));
}
__device__ __forceinline__ float ldg1(const float *p) { return __ldg(p); }

// ---- reductions into global memory (fire-and-forget) ----------------------------
__device__ __forceinline__ void red_add4(float *p, float4 v) {
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void red_add1(float *p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// Packed fp32 pairs (sm_100a FMUL2 / FADD2: two IEEE round-to-nearest fp32
// operations per lane in one issue slot; element results identical to
// FMUL / FADD).  Opt-in (-DSYSTEC_F32X2): measured, 18 % fewer instructions
// per entry change no symmetric kernel's time and make the naive baseline
// kernel 1.5 % (c2) to 5 % (c4) slower (profiles/r02/s4/f32x2_ab.txt), so the
// default build keeps the scalar forms.
#ifdef SYSTEC_F32X2
__device__ __forceinline__ void mul2(float &r0, float &r1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
        "mul.rn.f32x2 rc, ra, rb;\n\tmov.b64 {%0,%1}, rc;\n\t}"
        : "=f"(r0), "=f"(r1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void add2(float &r0, float &r1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
        "add.rn.f32x2 rc, ra, rb;\n\tmov.b64 {%0,%1}, rc;\n\t}"
        : "=f"(r0), "=f"(r1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
#else
__device__ __forceinline__ void mul2(float &r0, float &r1, float a0, float a1, float b0, float b1) {
    r0 = a0 * b0;
    r1 = a1 * b1;
}
__device__ __forceinline__ void add2(float &r0, float &r1, float a0, float a1, float b0, float b1) {
    r0 = a0 + b0;
    r1 = a1 + b1;
}
#endif

// predicated forms: one REDG issued under a predicate, no branch
__device__ __forceinline__ void red_add4_if(float *p, float4 v, bool pred) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
        "@q red.global.add.v4.f32 [%0], {%1,%2,%3,%4};\n\t}" ::"l"(p),
        "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(static_cast<int>(pred))
        : "memory");
}
__device__ __forceinline__ void red_add1_if(float *p, float v, bool pred) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
        "@q red.global.add.f32 [%0], %1;\n\t}" ::"l"(p),
        "f"(v), "r"(static_cast<int>(pred))
        : "memory");
}

}  // namespace systec
