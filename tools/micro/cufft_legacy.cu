// cuFFT legacy (static-library) callback variant of cufft_lto.cu.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -rdc=true tools/micro/cufft_legacy.cu -lcufft_static -lculibos -o /tmp/leg
// cuFFT LTO-callback experiment for the camera-ID PCE (720x1280, batch 64):
// (a) template kernel + R2C + conj-mul kernel + C2R, vs (b) R2C with a load callback
// forming T = K * I and C2R with a load callback forming conj-mul + DC zero.
//   nvcc -gencode arch=compute_100a,code=lto_100a -rdc=true -fatbin tools/micro/cufft_lto_cb.cu -o /tmp/cb.fatbin
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/micro/cufft_lto.cu -lcufft -o /tmp/lto && /tmp/lto /tmp/cb.fatbin
#include <cufftXt.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <chrono>
#define CK(x) do { auto e_ = (x); if (e_) { printf("%s:%d err %d\n", __FILE__, __LINE__, (int)e_); exit(1); } } while (0)
struct TplInfo { const float* K; const uint8_t* I; unsigned long long P; };
struct MulInfo { const cufftComplex* R; unsigned long long n_per; };

__global__ void k_tpl(const float* K, const uint8_t* I, long long P, int b, float* T) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < P * b; i += 256LL * gridDim.x) T[i] = K[i % P] * (float)I[i];
}
__global__ void k_mul(const cufftComplex* R, cufftComplex* T, long long n_per, long long n) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) {
        cufftComplex r = R[i], t = T[i], o;
        o.x = r.x * t.x + r.y * t.y;
        o.y = r.y * t.x - r.x * t.y;
        if (i % n_per == 0) o.x = o.y = 0.f;
        T[i] = o;
    }
}
__global__ void k_init(float* x, long long n, unsigned s) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) {
        unsigned h = (unsigned)i * 2654435761u ^ s; h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
        x[i] = (h & 0xffff) / 65536.0f - 0.5f;
    }
}
__global__ void k_init8(uint8_t* x, long long n) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) x[i] = (uint8_t)((i * 7919) % 251);
}

__device__ cufftReal tpl_load(void* in, size_t off, void* ci, void* sh) {
    const TplInfo* t = (const TplInfo*)ci;
    return t->K[off % t->P] * (float)t->I[off];
}
__device__ cufftComplex mul_load(void* in, size_t off, void* ci, void* sh) {
    const MulInfo* m = (const MulInfo*)ci;
    cufftComplex r = m->R[off], t = ((const cufftComplex*)in)[off], o;
    o.x = r.x * t.x + r.y * t.y;
    o.y = r.y * t.x - r.x * t.y;
    if (off % m->n_per == 0) o.x = o.y = 0.f;
    return o;
}
__device__ cufftCallbackLoadR d_tpl = tpl_load;
__device__ cufftCallbackLoadC d_mul = mul_load;

int main(int argc, char** argv) {
    const int H = 720, W = 1280, B = 64;
    const long long P = (long long)H * W, NS = (long long)H * (W / 2 + 1);
    float *K, *T, *C0, *C1, *Rr; uint8_t* I; cufftComplex *Rs, *S;
    CK(cudaMalloc(&K, P * 4)); CK(cudaMalloc(&T, P * B * 4)); CK(cudaMalloc(&C0, P * B * 4)); CK(cudaMalloc(&C1, P * B * 4));
    CK(cudaMalloc(&Rr, P * B * 4)); CK(cudaMalloc(&I, P * B)); CK(cudaMalloc(&Rs, NS * B * 8)); CK(cudaMalloc(&S, NS * B * 8));
    k_init<<<1184, 256>>>(K, P, 1); k_init<<<1184, 256>>>(Rr, P * B, 2); k_init8<<<1184, 256>>>(I, P * B);
    int n[2] = {H, W};
    cufftHandle r2c, c2r, r2c_cb, c2r_cb; 
    CK(cufftPlanMany(&r2c, 2, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_R2C, B));
    CK(cufftPlanMany(&c2r, 2, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_C2R, B));
    CK(cufftExecR2C(r2c, Rr, Rs));   // residual spectrum
    TplInfo ti{K, I, (unsigned long long)P}; MulInfo mi{Rs, (unsigned long long)NS};
    TplInfo* dti; MulInfo* dmi;
    CK(cudaMalloc(&dti, sizeof ti)); CK(cudaMalloc(&dmi, sizeof mi));
    CK(cudaMemcpy(dti, &ti, sizeof ti, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dmi, &mi, sizeof mi, cudaMemcpyHostToDevice));
    auto t0 = std::chrono::steady_clock::now();
    void *h_tpl, *h_mul;
    CK(cudaMemcpyFromSymbol(&h_tpl, d_tpl, sizeof(void*)));
    CK(cudaMemcpyFromSymbol(&h_mul, d_mul, sizeof(void*)));
    CK(cufftPlanMany(&r2c_cb, 2, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_R2C, B));
    CK(cufftXtSetCallback(r2c_cb, &h_tpl, CUFFT_CB_LD_REAL, (void**)&dti));
    CK(cufftPlanMany(&c2r_cb, 2, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_C2R, B));
    CK(cufftXtSetCallback(c2r_cb, &h_mul, CUFFT_CB_LD_COMPLEX, (void**)&dmi));
    auto t1 = std::chrono::steady_clock::now();
    printf("callback plan creation %.1f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count());
    auto base = [&] {
        k_tpl<<<1184, 256>>>(K, I, P, B, T);
        cufftExecR2C(r2c, T, S);
        k_mul<<<1184, 256>>>(Rs, S, NS, NS * B);
        cufftExecC2R(c2r, S, C0);
    };
    auto cb = [&] {
        cufftExecR2C(r2c_cb, T, S);
        cufftExecC2R(c2r_cb, S, C1);
    };
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int v = 0; v < 2; ++v) {
        for (int w = 0; w < 3; ++w) v ? cb() : base();
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) v ? cb() : base();
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%s: %.3f ms per 64-pair batch\n", v ? "callbacks" : "baseline ", ms / 20);
    }
    CK(cudaGetLastError());
    std::vector<float> a(P * B), b(P * B);
    cudaMemcpy(a.data(), C0, P * B * 4, cudaMemcpyDeviceToHost); cudaMemcpy(b.data(), C1, P * B * 4, cudaMemcpyDeviceToHost);
    double md = 0, mx = 0;
    for (long long i = 0; i < P * B; ++i) { md = fmax(md, fabs(a[i] - b[i])); mx = fmax(mx, fabs(a[i])); }
    printf("max |C_base - C_cb| = %.3g (max |C| %.3g)\n", md, mx);
    return 0;
}
