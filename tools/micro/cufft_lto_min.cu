// Minimal cuFFT LTO-callback probe: 1-D C2C / R2C of length N, batch B, load callback.
#include <cufftXt.h>
#include <cstdio>
#include <vector>
int main(int argc, char** argv) {
    FILE* f = fopen(argv[1], "rb");
    fseek(f, 0, SEEK_END); size_t fsz = ftell(f); fseek(f, 0, SEEK_SET);
    std::vector<char> fb(fsz);
    if (fread(fb.data(), 1, fsz, f) != fsz) return 1;
    fclose(f);
    int cases[][3] = {{1024, 1, 0}, {1024, 1, 1}, {1280, 1, 1}, {720, 2, 1}};
    for (auto& c : cases) {
        cufftHandle p;
        size_t ws;
        cufftCreate(&p);
        void* ci = nullptr;
        int n[2] = {c[1] == 2 ? 720 : c[0], 1280};
        cufftResult r1 = cufftXtSetJITCallback(p, c[2] ? "tpl_load" : "mul_load", fb.data(), fsz,
                                               c[2] ? CUFFT_CB_LD_REAL : CUFFT_CB_LD_COMPLEX, &ci);
        cufftResult r2 = cufftMakePlanMany(p, c[1], n, nullptr, 1, 0, nullptr, 1, 0, c[2] ? CUFFT_R2C : CUFFT_C2C, 4, &ws);
        printf("N=%d rank=%d %s: set %d make %d\n", c[0], c[1], c[2] ? "R2C" : "C2C", (int)r1, (int)r2);
        cufftDestroy(p);
    }
    return 0;
}
