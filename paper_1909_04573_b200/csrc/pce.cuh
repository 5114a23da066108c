// pce.cuh — PCE peak / energy partials shared by pce.cu and pcefft.cu (sm_100a).
#pragma once

#include "common.cuh"

namespace prnu {

struct PeakE {
    float a;      // |C| of the best candidate
    int idx;      // its linear index (-1 = none)
    double e;     // partial energy
};

__device__ __forceinline__ bool better(float a1, int i1, float a2, int i2) {
    // larger |C| wins; ties -> smaller index; idx -1 always loses
    if (i2 < 0) return i1 >= 0;
    if (i1 < 0) return false;
    return a1 > a2 || (a1 == a2 && i1 < i2);
}

// Offer candidate (a, i) to a thread's running best: larger |C| wins, ties -> the
// smaller index; NaN never becomes a candidate (a > best is false).
__device__ __forceinline__ void offer(float a, int i, float& best, int& bi) {
    if (a > best || (a == best && bi >= 0 && i < bi)) {
        best = a;
        bi = i;
    }
}

}  // namespace prnu
