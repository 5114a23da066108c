// Microbenchmark (sm_100a): shared-memory wavefronts of LDS.64 / LDS.128 warp
// accesses where lane l reads row (l & RMASK) at a row pitch P (floats) plus a
// column offset of (l >> RSHIFT) * CSTEP floats.  Run under ncu and compare
// l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld per kernel with the ideal.
#include <cstdio>
#include <cuda_runtime.h>
template <int W, int P, int RBITS, int CSTEP>
__global__ void k(float* out, int n) {
    __shared__ __align__(16) float s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i;
    __syncthreads();
    const int l = threadIdx.x & 31;
    const int row = l & ((1 << RBITS) - 1), col = (l >> RBITS) * CSTEP;
    const float* p = s + row * P + col;
    float acc = 0.f;
    for (int it = 0; it < n; ++it) {
        if (W == 4) { const float4 v = *reinterpret_cast<const float4*>(p + (it & 3) * 4); acc += v.x + v.y + v.z + v.w; }
        if (W == 2) { const float2 v = *reinterpret_cast<const float2*>(p + (it & 3) * 2); acc += v.x + v.y; }
        asm volatile("" ::: "memory");
    }
    if (acc == 1234.5f) out[threadIdx.x] = acc;
}
int main() {
    float* o;
    cudaMalloc(&o, 4096);
#define RUN(W, P, RB, CS) k<W, P, RB, CS><<<1, 32>>>(o, 64); printf("W%d P%d rows%d cstep%d\n", W, P, 1 << RB, CS);
    RUN(4, 124, 3, 8)   // the da H-pass pattern: 8 rows x 4 column groups of 8 floats
    RUN(4, 116, 3, 8)
    RUN(4, 132, 3, 8)
    RUN(4, 124, 3, 4)
    RUN(4, 124, 2, 8)
    RUN(4, 244, 3, 16)  // the pair H-pass pattern (float2 pitch 122)
    RUN(4, 228, 3, 16)
    RUN(4, 36, 4, 4)    // u8 row pass: 16 rows x 2 groups (words), pitch 36 words
    RUN(2, 36, 4, 4)
    RUN(2, 34, 4, 4)
    RUN(4, 128, 0, 4)   // contiguous (ideal 4 per request)
    cudaDeviceSynchronize();
    return 0;
}
