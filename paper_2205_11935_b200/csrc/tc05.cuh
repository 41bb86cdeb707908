// tc05.cuh -- sm_100a 5th-generation tensor-core primitives (tcgen05 MMA with TMEM accumulators, mbarriers)
// used by the exact modular contractions on the integer tensor path (k_mac_tc.cu).  Encodings follow the
// PTX ISA 8.7 descriptors (validated on the device by tools/tc_i8_test.cu: u8 x u8 -> s32, K-major,
// SWIZZLE_NONE canonical layouts, bit-exact against a CPU reference, 2.09 POPS = 93% of the nominal dense
// int8 rate at N >= 128).
#pragma once
#include <cstdint>

namespace ck {

__device__ __forceinline__ uint32_t tc_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMEM allocation by one full warp; the base address is written to shared memory
__device__ __forceinline__ void tc_tmem_alloc(uint32_t* dst_smem, uint32_t ncols)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tc_tmem_dealloc(uint32_t taddr, uint32_t ncols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t* bar, uint32_t phase)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "TC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TC_WAIT_%=;\n\t}" ::"r"(tc_smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// K-major SWIZZLE_NONE shared-memory matrix descriptor: core matrices of 8 rows x 16 bytes (128 B contiguous);
// lbo = byte distance between K-adjacent core matrices, sbo = between M/N-adjacent 8-row groups
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// kind::i8 instruction descriptor: D s32, A and B unsigned 8-bit, both K-major, M x N
__host__ __device__ constexpr uint32_t tc_idesc_u8(int M, int N)
{
    return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// D[tmem] (+)= A[smem] . B[smem]^T   (128 x N x 32 bytes), issued by one thread
__device__ __forceinline__ void tc_mma_u8(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// arrive on an mbarrier when every MMA issued so far by this thread has completed
__device__ __forceinline__ void tc_commit(uint64_t* bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        tc_smem_u32(bar)));
}
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void tc_fence_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
// 32 lanes x 16 consecutive 32-bit columns: lane (row) = warp's TMEM lane quarter + lane id
__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tc_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// byte-reversed, shifted key/plaintext word for the shift-class B operand (k_mac_tc.cu): the 8 bytes u = 0..7
// of the result hold byte (s - u) of w (0 outside 0..7), so that sum_u a_u b_u over a little-endian 64-bit A
// word a equals sum_{u + v = s} a_u w_v
__device__ __forceinline__ uint64_t tc_shift_bytes(uint64_t w, int s)
{
    const uint64_t x = s <= 7 ? (w << (8 * (7 - s))) : (w >> (8 * (s - 7)));
    const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    return ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | (uint64_t)__byte_perm(hi, 0, 0x0123);
}

}  // namespace ck
