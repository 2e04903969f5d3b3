// tc_ptx.cuh -- inline-PTX building blocks for the sm_100a tcgen05 kernels
// (mbarriers, 1-D bulk copies, tcgen05 MMA / commit / fences, TMEM loads).
// Shared by tensor_scan.cu (K3) and flashmatch.cu (K7); compile with
// -gencode arch=compute_100a,code=sm_100a.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fnl {
namespace {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_addr(bar);
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
// try_wait with a long suspend-time hint: the warp sleeps in hardware until
// the phase completes (or the hint expires) instead of re-polling, so helper
// warps (loader / MMA issuer) do not steal issue slots from co-resident
// epilogue warps on the same SM sub-partition
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_addr(bar);
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity), "r"(1000000u)
            : "memory");
    } while (!done);
}
// spin on mbarrier.test_wait (never suspends the warp): lower wake-up latency
// than try_wait when the phase completes within a few hundred cycles
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_addr(bar);
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(
            d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// D[tmem] (+)= A[tmem] . B[smem]^T  (A resident in tensor memory)
__device__ __forceinline__ void tc_mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(
            d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// 128 rows x 256 bits (one K=16 slice of an M=128 operand) smem -> TMEM
__device__ __forceinline__ void tc_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{ .reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0, 1, 0, p; }" : "=r"(pred));
    return pred != 0;
}

// tcgen05.ld of 32 columns whose destination registers are tied to the
// matching wait, so no use of them can be scheduled before tcgen05.wait::ld.
struct Frag {
    uint32_t r[32];
};
__device__ __forceinline__ void frag_ld(uint32_t taddr, Frag& f) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(f.r[0]), "=r"(f.r[1]), "=r"(f.r[2]), "=r"(f.r[3]), "=r"(f.r[4]), "=r"(f.r[5]), "=r"(f.r[6]),
          "=r"(f.r[7]), "=r"(f.r[8]), "=r"(f.r[9]), "=r"(f.r[10]), "=r"(f.r[11]), "=r"(f.r[12]),
          "=r"(f.r[13]), "=r"(f.r[14]), "=r"(f.r[15]), "=r"(f.r[16]), "=r"(f.r[17]), "=r"(f.r[18]),
          "=r"(f.r[19]), "=r"(f.r[20]), "=r"(f.r[21]), "=r"(f.r[22]), "=r"(f.r[23]), "=r"(f.r[24]),
          "=r"(f.r[25]), "=r"(f.r[26]), "=r"(f.r[27]), "=r"(f.r[28]), "=r"(f.r[29]), "=r"(f.r[30]),
          "=r"(f.r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void frag_wait1(Frag& f) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(f.r[0]), "+r"(f.r[1]), "+r"(f.r[2]), "+r"(f.r[3]), "+r"(f.r[4]), "+r"(f.r[5]),
                   "+r"(f.r[6]), "+r"(f.r[7]), "+r"(f.r[8]), "+r"(f.r[9]), "+r"(f.r[10]), "+r"(f.r[11]),
                   "+r"(f.r[12]), "+r"(f.r[13]), "+r"(f.r[14]), "+r"(f.r[15]), "+r"(f.r[16]), "+r"(f.r[17]),
                   "+r"(f.r[18]), "+r"(f.r[19]), "+r"(f.r[20]), "+r"(f.r[21]), "+r"(f.r[22]), "+r"(f.r[23]),
                   "+r"(f.r[24]), "+r"(f.r[25]), "+r"(f.r[26]), "+r"(f.r[27]), "+r"(f.r[28]), "+r"(f.r[29]),
                   "+r"(f.r[30]), "+r"(f.r[31])
                 :
                 : "memory");
}

// one tcgen05.ld of 64 consecutive columns (32x32b.x64) into two fragments
__device__ __forceinline__ void frag_ld64(uint32_t taddr, Frag& f, Frag& g) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(f.r[0]), "=r"(f.r[1]), "=r"(f.r[2]), "=r"(f.r[3]), "=r"(f.r[4]), "=r"(f.r[5]), "=r"(f.r[6]), "=r"(f.r[7]), "=r"(f.r[8]), "=r"(f.r[9]), "=r"(f.r[10]), "=r"(f.r[11]), "=r"(f.r[12]), "=r"(f.r[13]), "=r"(f.r[14]), "=r"(f.r[15]), "=r"(f.r[16]), "=r"(f.r[17]), "=r"(f.r[18]), "=r"(f.r[19]), "=r"(f.r[20]), "=r"(f.r[21]), "=r"(f.r[22]), "=r"(f.r[23]), "=r"(f.r[24]), "=r"(f.r[25]), "=r"(f.r[26]), "=r"(f.r[27]), "=r"(f.r[28]), "=r"(f.r[29]), "=r"(f.r[30]), "=r"(f.r[31]), "=r"(g.r[0]), "=r"(g.r[1]), "=r"(g.r[2]), "=r"(g.r[3]), "=r"(g.r[4]), "=r"(g.r[5]), "=r"(g.r[6]), "=r"(g.r[7]), "=r"(g.r[8]), "=r"(g.r[9]), "=r"(g.r[10]), "=r"(g.r[11]), "=r"(g.r[12]), "=r"(g.r[13]), "=r"(g.r[14]), "=r"(g.r[15]), "=r"(g.r[16]), "=r"(g.r[17]), "=r"(g.r[18]), "=r"(g.r[19]), "=r"(g.r[20]), "=r"(g.r[21]), "=r"(g.r[22]), "=r"(g.r[23]), "=r"(g.r[24]), "=r"(g.r[25]), "=r"(g.r[26]), "=r"(g.r[27]), "=r"(g.r[28]), "=r"(g.r[29]), "=r"(g.r[30]), "=r"(g.r[31])
        : "r"(taddr));
}
// one tcgen05.ld of 128 consecutive 16-bit-accumulator columns (32x32b.x64
// with .pack::16b: two adjacent columns per register) into two fragments
__device__ __forceinline__ void frag_ld128_p16(uint32_t taddr, Frag& f, Frag& g) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(f.r[0]), "=r"(f.r[1]), "=r"(f.r[2]), "=r"(f.r[3]), "=r"(f.r[4]), "=r"(f.r[5]), "=r"(f.r[6]), "=r"(f.r[7]), "=r"(f.r[8]), "=r"(f.r[9]), "=r"(f.r[10]), "=r"(f.r[11]), "=r"(f.r[12]), "=r"(f.r[13]), "=r"(f.r[14]), "=r"(f.r[15]), "=r"(f.r[16]), "=r"(f.r[17]), "=r"(f.r[18]), "=r"(f.r[19]), "=r"(f.r[20]), "=r"(f.r[21]), "=r"(f.r[22]), "=r"(f.r[23]), "=r"(f.r[24]), "=r"(f.r[25]), "=r"(f.r[26]), "=r"(f.r[27]), "=r"(f.r[28]), "=r"(f.r[29]), "=r"(f.r[30]), "=r"(f.r[31]), "=r"(g.r[0]), "=r"(g.r[1]), "=r"(g.r[2]), "=r"(g.r[3]), "=r"(g.r[4]), "=r"(g.r[5]), "=r"(g.r[6]), "=r"(g.r[7]), "=r"(g.r[8]), "=r"(g.r[9]), "=r"(g.r[10]), "=r"(g.r[11]), "=r"(g.r[12]), "=r"(g.r[13]), "=r"(g.r[14]), "=r"(g.r[15]), "=r"(g.r[16]), "=r"(g.r[17]), "=r"(g.r[18]), "=r"(g.r[19]), "=r"(g.r[20]), "=r"(g.r[21]), "=r"(g.r[22]), "=r"(g.r[23]), "=r"(g.r[24]), "=r"(g.r[25]), "=r"(g.r[26]), "=r"(g.r[27]), "=r"(g.r[28]), "=r"(g.r[29]), "=r"(g.r[30]), "=r"(g.r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void frag_wait2(Frag& f, Frag& g) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(f.r[0]), "+r"(f.r[1]), "+r"(f.r[2]), "+r"(f.r[3]), "+r"(f.r[4]), "+r"(f.r[5]),
                   "+r"(f.r[6]), "+r"(f.r[7]), "+r"(f.r[8]), "+r"(f.r[9]), "+r"(f.r[10]), "+r"(f.r[11]),
                   "+r"(f.r[12]), "+r"(f.r[13]), "+r"(f.r[14]), "+r"(f.r[15]), "+r"(f.r[16]), "+r"(f.r[17]),
                   "+r"(f.r[18]), "+r"(f.r[19]), "+r"(f.r[20]), "+r"(f.r[21]), "+r"(f.r[22]), "+r"(f.r[23]),
                   "+r"(f.r[24]), "+r"(f.r[25]), "+r"(f.r[26]), "+r"(f.r[27]), "+r"(f.r[28]), "+r"(f.r[29]),
                   "+r"(f.r[30]), "+r"(f.r[31]), "+r"(g.r[0]), "+r"(g.r[1]), "+r"(g.r[2]), "+r"(g.r[3]),
                   "+r"(g.r[4]), "+r"(g.r[5]), "+r"(g.r[6]), "+r"(g.r[7]), "+r"(g.r[8]), "+r"(g.r[9]),
                   "+r"(g.r[10]), "+r"(g.r[11]), "+r"(g.r[12]), "+r"(g.r[13]), "+r"(g.r[14]), "+r"(g.r[15]),
                   "+r"(g.r[16]), "+r"(g.r[17]), "+r"(g.r[18]), "+r"(g.r[19]), "+r"(g.r[20]), "+r"(g.r[21]),
                   "+r"(g.r[22]), "+r"(g.r[23]), "+r"(g.r[24]), "+r"(g.r[25]), "+r"(g.r[26]), "+r"(g.r[27]),
                   "+r"(g.r[28]), "+r"(g.r[29]), "+r"(g.r[30]), "+r"(g.r[31])
                 :
                 : "memory");
}

}  // namespace
}  // namespace fnl
