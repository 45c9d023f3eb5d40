// PCG64 (numpy's XSL-RR 128/64) with O(log k) jump-ahead, shared by the
// device generators (countsketch.cu: K1, omega.cu: Gaussian test matrix).
//
// x' = M x + inc on 128-bit state; k steps compose to x_k = M^k x + inc * G_k
// with G_k = sum_{i<k} M^i.  Draw d (0-based) is the output of the state
// after d + 1 steps: xsl_rr(apply(affine(jpow(d + 1), inc), state)).
#pragma once
#include <stdint.h>

namespace skp {
namespace {

typedef unsigned __int128 u128;

__host__ __device__ inline u128 mk128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

struct Jump {  // k steps: x -> m * x + g * inc
    u128 m, g;
};

__host__ __device__ inline u128 pcg_mult() {
    return mk128(2549297995355413924ULL, 4865540595714422341ULL);
}

__host__ __device__ inline Jump jcompose(Jump a, Jump b) {  // a then b (commutative)
    Jump r;
    r.m = a.m * b.m;
    r.g = b.m * a.g + b.g;
    return r;
}

__host__ __device__ inline Jump jpow(uint64_t k) {
    Jump acc{1, 0}, cur{pcg_mult(), 1};
    while (k) {
        if (k & 1) acc = jcompose(acc, cur);
        cur = jcompose(cur, cur);
        k >>= 1;
    }
    return acc;
}

struct Affine {  // precombined with inc: x -> m * x + c
    u128 m, c;
};
__host__ __device__ inline Affine affine(Jump j, u128 inc) { return Affine{j.m, j.g * inc}; }
__host__ __device__ inline u128 apply(Affine a, u128 x) { return a.m * x + a.c; }

__device__ __forceinline__ uint64_t xsl_rr(u128 x) {
    uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
    unsigned rot = (unsigned)(hi >> 58);
    uint64_t v = hi ^ lo;
    return (v >> rot) | (v << ((64u - rot) & 63u));
}

}  // namespace
}  // namespace skp
