// TMA staging of column-major fp64 row windows (sm_100a).  Product code.
//
// A rank's A (m rows x n columns, column-major, leading dimension lda) is
// described by one 2-D tensor map: dim 0 = rows (contiguous), dim 1 = columns
// (stride lda * 8 bytes).  A box of `box_rows` x `box_cols` lands in shared
// memory column-major ([col][row], rows contiguous), exactly the staging
// layout the chunk kernels read; rows >= m and columns >= n are zero-filled
// by the hardware.  One elected lane issues the copy; completion is an
// mbarrier transaction count (mbarrier.try_wait.parity).
//
// Host side: make_tmap_colmajor() returns false when TMA cannot describe the
// matrix (base not 16-byte aligned, lda * 8 not a multiple of 16, more than
// 2^31 rows); the kernels then keep the per-element cp.async path.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tsqr {
namespace tma {

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// generic-proxy accesses of this thread's earlier smem reads/writes ordered
// before later async-proxy (TMA) accesses to the same buffer
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

// box (row0 .. row0 + box_rows, col0 .. col0 + box_cols) -> smem dst (16-byte aligned)
__device__ __forceinline__ void load_2d(void *dst, const CUtensorMap *map, int row0, int col0, uint64_t *bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(d),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(row0), "r"(col0), "r"(b)
        : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace tma

// Host: tensor map of an m x n column-major fp64 matrix with box (box_rows, box_cols).
bool make_tmap_colmajor(CUtensorMap *map, const double *base, int64_t m, int64_t n, int64_t ld, int box_rows,
                        int box_cols);

}  // namespace tsqr
