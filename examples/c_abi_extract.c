/* c_abi_extract.c — the fingerprint path driven from plain C through include/prnu.h
 * (no Python, no torch): read a u8 frame stack from a file, extract the SDA
 * fingerprint on the GPU, write K (fp32) and the NCC of K with a second K file.
 *
 *   c_abi_extract frames.u8 m H W depth K_out.f32 [K_ref.f32]
 *
 * Build: gcc -O2 -I include examples/c_abi_extract.c -L paper_1909_04573_b200 -lprnu
 *        -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,... (tests/test_gpu_c_abi.py) */
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <cuda_runtime_api.h>
#include "prnu.h"

#define CK(x)                                                                   \
    do {                                                                        \
        int rc_ = (x);                                                          \
        if (rc_) {                                                              \
            fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, prnu_last_error()); \
            return 1;                                                           \
        }                                                                       \
    } while (0)
#define CU(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));            \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

static void* read_file(const char* path, size_t bytes) {
    FILE* f = fopen(path, "rb");
    if (!f) return NULL;
    void* p = malloc(bytes);
    if (p && fread(p, 1, bytes, f) != bytes) {
        free(p);
        p = NULL;
    }
    fclose(f);
    return p;
}

int main(int argc, char** argv) {
    if (argc < 7) {
        fprintf(stderr, "usage: %s frames.u8 m H W depth K_out.f32 [K_ref.f32]\n", argv[0]);
        return 2;
    }
    const int64_t m = atoll(argv[2]), depth = atoll(argv[5]);
    const int H = atoi(argv[3]), W = atoi(argv[4]);
    const size_t P = (size_t)H * W;
    uint8_t* frames_h = (uint8_t*)read_file(argv[1], (size_t)m * P);
    if (!frames_h) {
        fprintf(stderr, "cannot read %s\n", argv[1]);
        return 1;
    }
    prnu_denoise_params p;
    CK(prnu_default_params(&p));
    const int batch = 16;
    const size_t ws_bytes = prnu_extract_workspace_bytes(H, W, batch, depth, &p);
    if (!ws_bytes) {
        fprintf(stderr, "invalid extraction arguments\n");
        return 1;
    }
    uint8_t* frames;
    float* K;
    double *sum_wi, *sum_i2;
    void* ws;
    CU(cudaMalloc((void**)&frames, (size_t)m * P));
    CU(cudaMalloc((void**)&K, sizeof(float) * P));
    CU(cudaMalloc((void**)&sum_wi, sizeof(double) * P));
    CU(cudaMalloc((void**)&sum_i2, sizeof(double) * P));
    CU(cudaMalloc(&ws, ws_bytes));
    CU(cudaMemcpy(frames, frames_h, (size_t)m * P, cudaMemcpyHostToDevice));
    int64_t n_sda = 0;
    CK(prnu_extract_fingerprint(frames, m, H, W, depth, &p, batch, 1e-6, K, sum_wi, sum_i2, &n_sda, ws, ws_bytes,
                                NULL));
    float* K_h = (float*)malloc(sizeof(float) * P);
    CU(cudaMemcpy(K_h, K, sizeof(float) * P, cudaMemcpyDeviceToHost));
    FILE* fo = fopen(argv[6], "wb");
    if (!fo || fwrite(K_h, sizeof(float), P, fo) != P) {
        fprintf(stderr, "cannot write %s\n", argv[6]);
        return 1;
    }
    fclose(fo);
    printf("n_sda %lld\n", (long long)n_sda);
    if (argc > 7) {   /* NCC of K with a reference fingerprint, on the GPU */
        float* ref_h = (float*)read_file(argv[7], sizeof(float) * P);
        if (!ref_h) return 1;
        float* ref;
        double* rho;
        CU(cudaMalloc((void**)&ref, sizeof(float) * P));
        CU(cudaMalloc((void**)&rho, sizeof(double)));
        CU(cudaMemcpy(ref, ref_h, sizeof(float) * P, cudaMemcpyHostToDevice));
        const size_t nws = prnu_ncc_workspace_bytes(1, H, W);
        void* nw;
        CU(cudaMalloc(&nw, nws));
        CK(prnu_ncc(K, ref, 1, H, W, rho, nw, nws, NULL));
        double rho_h;
        CU(cudaMemcpy(&rho_h, rho, sizeof(double), cudaMemcpyDeviceToHost));
        printf("ncc %.17g\n", rho_h);
    }
    printf("launches %llu\n", (unsigned long long)prnu_kernel_launches());
    return 0;
}
