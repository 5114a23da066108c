#include <cufftXt.h>
#include <cstdint>
struct TplInfo { const float* K; const uint8_t* I; unsigned long long P; };
struct MulInfo { const cufftComplex* R; unsigned long long n_per; };
extern "C" __device__ cufftReal tpl_load(void* in, unsigned long long off, void* ci, void* sh) {
    const TplInfo* t = (const TplInfo*)ci;
    return t->K[off % t->P] * (float)t->I[off];
}
extern "C" __device__ cufftComplex mul_load(void* in, unsigned long long off, void* ci, void* sh) {
    const MulInfo* m = (const MulInfo*)ci;
    cufftComplex r = m->R[off], t = ((const cufftComplex*)in)[off], o;
    o.x = r.x * t.x + r.y * t.y;
    o.y = r.y * t.x - r.x * t.y;
    if (off % m->n_per == 0) o.x = o.y = 0.f;
    return o;
}
