// Standalone probe of 3-D TMA box loads: tma_u8_test <dtype u8|f32> <box_w> <box_h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../paper_1909_04573_b200/csrc/tma.cuh"

__global__ void k(const __grid_constant__ CUtensorMap m, int bytes, int x, int y, unsigned char* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + ((bytes + 127) / 128) * 128);
    if (threadIdx.x == 0) { prnu::mbar_init(bar, 1); prnu::fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) { prnu::mbar_arrive_expect_tx(bar, bytes); prnu::tma_load_3d(sm, &m, x, y, 0, bar); }
    prnu::mbar_wait(bar, 0);
    for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
    bool u8 = !strcmp(argv[1], "u8");
    int bw = atoi(argv[2]), bh = atoi(argv[3]);
    int es = u8 ? 1 : 4;
    const int W = 1920, H = 1080;
    void* d; cudaMalloc(&d, (size_t)W * H * 2 * es);
    unsigned char* o; cudaMalloc(&o, 1 << 22);
    PFN_cuTensorMapEncodeTiled_v12000 fn; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 2};
    cuuint64_t str[2] = {(cuuint64_t)W * es, (cuuint64_t)W * H * es};
    cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1}, est[3] = {1, 1, 1};
    CUresult r = fn(&m, u8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, est,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("%s bw %d bh %d encode fail %d\n", argv[1], bw, bh, (int)r); return 0; }
    int bytes = bw * bh * es;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    int x0 = argc > 4 ? atoi(argv[4]) : 100;
    k<<<1, 128, ((bytes + 127) / 128) * 128 + 16>>>(m, bytes, x0, 50, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s bw %3d bh %3d x0 %d -> %s\n", argv[1], bw, bh, x0, cudaGetErrorString(e));
    return 0;
}
