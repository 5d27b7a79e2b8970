// Software grid barrier and SM-spread CTA ranks for the persistent
// cooperative CG kernels (kernels_cg.cu, kernels_cg_res.cu).
#pragma once
#include <cuda_runtime.h>

#include "tile_gemm.cuh"

namespace cpkit {
namespace gsync {

// Grid barrier on a monotonically increasing arrival counter: one
// release-add per CTA, then acquire-polls until every CTA of this round has
// arrived (no reset, no generation word, no full fences).
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks, unsigned int& round) {
    __syncthreads();
    ++round;
    if (threadIdx.x == 0) {
        const unsigned int target = round * nblocks;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned int seen;
        for (unsigned long long spin = 0;; ++spin) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
            if (static_cast<int>(seen - target) >= 0) break;
            if (spin > (1ull << 30)) __trap();  // never hang the GPU on a lost arrival
        }
    }
    __syncthreads();
    tile::fence_async_global();  // later bulk copies (async proxy) see the data released by other CTAs
}

// The same barrier in two halves, for work that depends on no other CTA's
// data and can run while the slowest CTA is still on its way: arrive (release
// this CTA's earlier global writes), independent work, then wait.
__device__ __forceinline__ void grid_arrive(unsigned int* bar, unsigned int& round) {
    __syncthreads();
    ++round;
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}
__device__ __forceinline__ void grid_wait(unsigned int* bar, unsigned int nblocks, unsigned int round) {
    if (threadIdx.x == 0) {
        const unsigned int target = round * nblocks;
        unsigned int seen;
        for (unsigned long long spin = 0;; ++spin) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
            if (static_cast<int>(seen - target) >= 0) break;
            if (spin > (1ull << 30)) __trap();
        }
    }
    __syncthreads();
    tile::fence_async_global();
}

// Task-order rank: the hardware packs consecutive block indices onto the same
// SMs, so phases with fewer tasks than CTAs would double up on half the SMs.
// Rank CTAs by their slot on their SM first (slot-0 CTAs get ranks 0.., the
// others ranks grid-1 downwards), so tasks 0..#SMs-1 land on distinct SMs.
__device__ __forceinline__ int cta_rank(unsigned int* words) {
    __shared__ int rank;
    if (threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        const unsigned slot = atomicAdd(words + 4 + (smid & 1023u), 1u);
        rank = slot == 0 ? static_cast<int>(atomicAdd(words + 1, 1u))
                         : static_cast<int>(gridDim.x) - 1 - static_cast<int>(atomicAdd(words + 2, 1u));
    }
    __syncthreads();
    return rank;
}


}  // namespace gsync
}  // namespace cpkit
