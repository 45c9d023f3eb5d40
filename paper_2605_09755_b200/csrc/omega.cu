// The Gaussian test matrix Omega on the device: standard normals identical to
// numpy's Generator(PCG64).standard_normal((rows, cols)) / sqrt(cols)
// (reference power.py:137-138 via sketching.py's generator), optionally cast
// to fp32 like `.astype(np.float32)`.
//
// numpy draws normals with a 256-layer ziggurat (Marsaglia & Tsang; constants
// in ziggurat_tables.h, recovered from numpy by scripts/gen_ziggurat.py): one
// 64-bit draw per sample 98.8% of the time, one more draw for a wedge test
// (exp), or 2k more for Marsaglia's tail (log1p).  Which draw starts which
// sample is therefore data-dependent -- a chain through the stream.  Here:
//   1. attempt kernel: for EVERY stream position p, the outcome of a sample
//      attempt starting at p (value or rejection, and how many draws it uses),
//      16 positions per thread after one PCG64 jump-ahead;
//   2. unit walks: the stream is cut into units of kZU positions; for each of
//      kZE possible entry offsets a lane walks the attempt chain through its
//      unit and records (exit offset into the next unit, #values);
//   3. the unit maps are composed (groups of 32 units per warp, then one warp
//      over the groups) to the true entry and output offset of every unit;
//   4. write kernel: each unit walks from its true entry and writes values.
// Exactness: attempts use numpy's operation order without FMA contraction
// (explicit __d*_rn).  The wedge decision compares with CUDA's exp (<= 1 ulp
// from glibc's), so it can only differ when the two land on opposite sides of
// the threshold -- probability ~2^-52 per wedge test; tail values use CUDA's
// log1p and may differ from glibc's by 1 ulp in rare cases without shifting
// the stream.  tests pin the output against numpy directly.
#include "common.cuh"
#include "pcg.cuh"
#include "ziggurat_tables.h"

namespace skp {
namespace {

constexpr int kZU = 1024;         // stream positions per walk unit
constexpr int kZE = 32;           // entry offsets tracked per unit (one warp)
constexpr int kZPer = 16;         // positions per thread in the attempt kernel
constexpr int kZGroup = 32;       // units composed per warp
constexpr uint8_t kZValid = 0x80; // len byte: bit 7 = the attempt yields a value
constexpr unsigned long long kOmegaFailMark = 1ull << 50;

__device__ __forceinline__ double zig_u53(uint64_t d) {
    return (double)(d >> 11) * 0x1.0p-53;  // numpy next_double
}

struct Stream {
    u128 x;
    Affine one;
    __device__ __forceinline__ uint64_t next() {
        x = apply(one, x);
        return xsl_rr(x);
    }
};

// attempt outcome for every stream position: len[p] (| kZValid), val[p]
__global__ void zig_attempt_kernel(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi,
                                   uint64_t inc_lo, int64_t npos, uint8_t* __restrict__ len,
                                   double* __restrict__ val, int* __restrict__ fail) {
    const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kZPer;
    if (p0 >= npos) return;
    const u128 inc = mk128(inc_hi, inc_lo);
    const Stream s0{apply(affine(jpow((uint64_t)p0), inc), mk128(st_hi, st_lo)),
                    Affine{pcg_mult(), inc}};
    Stream s = s0;
    uint64_t d[kZPer];
#pragma unroll
    for (int i = 0; i < kZPer; ++i) d[i] = s.next();
#pragma unroll
    for (int i = 0; i < kZPer; ++i) {
        const int64_t p = p0 + i;
        if (p >= npos) break;
        const uint64_t r = d[i];
        const int idx = (int)(r & 0xff);
        const uint64_t rest = r >> 8;
        const uint64_t rabs = (rest >> 1) & 0x000fffffffffffffull;
        double x = __dmul_rn((double)rabs, kZigW[idx]);
        if (rest & 1) x = -x;
        if (rabs < kZigK[idx]) {
            len[p] = kZValid | 1;
            val[p] = x;
            continue;
        }
        // rare path: auxiliary draws p+1, p+2, ... from a stream re-derived
        // from the window start (no dynamic indexing of d[])
        Stream la = s0;
        for (int t = 0; t <= i; ++t) la.next();
        if (idx != 0) {
            const double u = zig_u53(la.next());
            const double lhs =
                __dadd_rn(__dmul_rn(__dsub_rn(kZigF[idx - 1], kZigF[idx]), u), kZigF[idx]);
            const double rhs = exp(__dmul_rn(__dmul_rn(-0.5, x), x));
            len[p] = (uint8_t)((lhs < rhs ? kZValid : 0) | 2);
            val[p] = x;
            continue;
        }
        int used = 1;
        for (;;) {
            const double xx = __dmul_rn(-kZigInvR, log1p(-zig_u53(la.next())));
            const double yy = -log1p(-zig_u53(la.next()));
            used += 2;
            if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
                const double t = __dadd_rn(kZigR, xx);
                val[p] = ((rabs >> 8) & 1) ? -t : t;
                break;
            }
            if (used > 0x7f - 2) {  // a tail longer than the len byte can hold
                atomicOr(fail, 1);
                break;
            }
        }
        len[p] = (uint8_t)(kZValid | (used > 0x7f ? 0x7f : used));
    }
}

// per unit and entry offset e: walk the chain -> (exit offset, #values)
__global__ void zig_walk_kernel(const uint8_t* __restrict__ len, int64_t nunits,
                                uint8_t* __restrict__ exitmap, uint16_t* __restrict__ cnt) {
    __shared__ uint8_t ls[kZU];
    const int64_t u = blockIdx.x;
    if (u >= nunits) return;
    for (int i = threadIdx.x; i < kZU; i += blockDim.x) ls[i] = len[u * kZU + i];
    __syncthreads();
    const int e = threadIdx.x;
    int p = e, c = 0;
    while (p < kZU) {
        const uint8_t l = ls[p];
        c += l >> 7;
        p += l & 0x7f;
    }
    const int ex = p - kZU;
    exitmap[u * kZE + e] = (uint8_t)(ex < kZE ? ex : 0xff);
    cnt[u * kZE + e] = (uint16_t)c;
}

// compose the maps of kZGroup consecutive units (lane = group entry offset)
__global__ void zig_group_kernel(const uint8_t* __restrict__ exitmap,
                                 const uint16_t* __restrict__ cnt, int64_t nunits,
                                 uint8_t* __restrict__ gexit, int32_t* __restrict__ gcnt) {
    const int64_t g = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int e = threadIdx.x & 31;
    const int64_t u0 = g * kZGroup;
    if (u0 >= nunits) return;
    int cur = e, tot = 0;
    for (int64_t u = u0; u < u0 + kZGroup && u < nunits; ++u) {
        if (cur == 0xff) break;
        tot += cnt[u * kZE + cur];
        cur = exitmap[u * kZE + cur];
    }
    gexit[g * kZE + e] = (uint8_t)cur;
    gcnt[g * kZE + e] = tot;
}

// one thread: the true entry / output offset of every group; flags overflow
// and a stream too short for `need` values
__global__ void zig_scan_groups_kernel(const uint8_t* __restrict__ gexit,
                                       const int32_t* __restrict__ gcnt, int64_t ngroups,
                                       int64_t need, uint8_t* __restrict__ gentry,
                                       int64_t* __restrict__ goff, int* __restrict__ fail) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int cur = 0;
    int64_t off = 0;
    for (int64_t g = 0; g < ngroups; ++g) {
        if (cur == 0xff) {
            atomicOr(fail, 2);
            return;
        }
        gentry[g] = (uint8_t)cur;
        goff[g] = off;
        off += gcnt[g * kZE + cur];
        cur = gexit[g * kZE + cur];
    }
    if (off < need) atomicOr(fail, 4);
}

// per group (one thread): entries / offsets of its units; then per unit the
// values are written by zig_write_kernel
__global__ void zig_units_kernel(const uint8_t* __restrict__ exitmap,
                                 const uint16_t* __restrict__ cnt, int64_t nunits,
                                 int64_t ngroups, const uint8_t* __restrict__ gentry,
                                 const int64_t* __restrict__ goff,
                                 uint8_t* __restrict__ uentry, int64_t* __restrict__ uoff) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    int cur = gentry[g];
    int64_t off = goff[g];
    for (int64_t u = g * kZGroup; u < (g + 1) * kZGroup && u < nunits; ++u) {
        uentry[u] = (uint8_t)cur;
        uoff[u] = off;
        if (cur == 0xff) continue;
        off += cnt[u * kZE + cur];
        cur = exitmap[u * kZE + cur];
    }
}

// one block per unit: stage the unit's attempts in smem, one thread walks the
// chain and marks value positions with their output index, all threads write
template <typename T>
__global__ void __launch_bounds__(256)
zig_write_kernel(const uint8_t* __restrict__ len, const double* __restrict__ val, int64_t nunits,
                 const uint8_t* __restrict__ uentry, const int64_t* __restrict__ uoff,
                 int64_t rows, int64_t cols, double divisor, T* __restrict__ out, int64_t ldo,
                 const int* __restrict__ fail) {
    __shared__ uint8_t ls[kZU];
    __shared__ int32_t slot[kZU];  // output index - uoff, or -1 (not a chain value)
    const int64_t u = blockIdx.x;
    if (u >= nunits || *fail) return;
    for (int i = threadIdx.x; i < kZU; i += blockDim.x) {
        ls[i] = len[u * kZU + i];
        slot[i] = -1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int p = uentry[u], k = 0;
        while (p < kZU) {
            const uint8_t l = ls[p];
            if (l & kZValid) slot[p] = k++;
            p += l & 0x7f;
        }
    }
    __syncthreads();
    const int64_t need = rows * cols, base = uoff[u];
    for (int i = threadIdx.x; i < kZU; i += blockDim.x) {
        const int s = slot[i];
        if (s < 0) continue;
        const int64_t k = base + s;
        if (k >= need) continue;
        const int64_t r = k / cols, c = k - r * cols;
        out[r * ldo + c] = (T)__ddiv_rn(val[u * kZU + i], divisor);
    }
}

// a failed generation poisons nothing silently: the caller's counter gets a mark
__global__ void zig_report_kernel(const int* __restrict__ fail, int64_t* counter) {
    if (*fail && counter) atomicAdd(reinterpret_cast<unsigned long long*>(counter), kOmegaFailMark);
}

struct ZigWs {
    int64_t npos, nunits, ngroups;
    uint8_t* len;
    double* val;
    uint8_t* exitmap;
    uint16_t* cnt;
    uint8_t* gexit;
    int32_t* gcnt;
    uint8_t* gentry;
    int64_t* goff;
    uint8_t* uentry;
    int64_t* uoff;
    int* fail;
    int64_t bytes;
};

ZigWs zig_layout(int64_t count, char* base) {
    ZigWs w;
    // ~1.2% of attempts reject, tails use extra draws: 1/32 headroom + slack
    const int64_t want = count + count / 32 + 4096;
    w.nunits = cdiv(want, (int64_t)kZU);
    w.npos = w.nunits * kZU;
    w.ngroups = cdiv(w.nunits, (int64_t)kZGroup);
    int64_t off = 0;
    auto take = [&](int64_t b) {
        char* p = base ? base + off : nullptr;
        off += (b + 255) / 256 * 256;
        return p;
    };
    w.val = reinterpret_cast<double*>(take(w.npos * 8));
    w.len = reinterpret_cast<uint8_t*>(take(w.npos));
    w.exitmap = reinterpret_cast<uint8_t*>(take(w.nunits * kZE));
    w.cnt = reinterpret_cast<uint16_t*>(take(w.nunits * kZE * 2));
    w.gexit = reinterpret_cast<uint8_t*>(take(w.ngroups * kZE));
    w.gcnt = reinterpret_cast<int32_t*>(take(w.ngroups * kZE * 4));
    w.gentry = reinterpret_cast<uint8_t*>(take(w.ngroups));
    w.goff = reinterpret_cast<int64_t*>(take(w.ngroups * 8));
    w.uentry = reinterpret_cast<uint8_t*>(take(w.nunits));
    w.uoff = reinterpret_cast<int64_t*>(take(w.nunits * 8));
    w.fail = reinterpret_cast<int*>(take(16));
    w.bytes = off;
    return w;
}

template <typename T>
int gaussian(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t rows,
             int64_t cols, double divisor, T* out, int64_t ldo, int64_t* fail_counter, void* ws,
             int64_t ws_bytes, cudaStream_t st) {
    SKP_ARG(rows >= 0 && cols >= 0 && ldo >= cols, "gaussian: bad sizes");
    const int64_t count = rows * cols;
    if (count == 0) return SKP_OK;
    ZigWs w = zig_layout(count, reinterpret_cast<char*>(ws));
    SKP_ARG(ws && ws_bytes >= w.bytes, "gaussian: needs %lld bytes of workspace",
            (long long)w.bytes);
    SKP_CUDA(cudaMemsetAsync(w.fail, 0, sizeof(int), st));
    const int64_t threads = cdiv(w.npos, (int64_t)kZPer);
    zig_attempt_kernel<<<(unsigned)cdiv(threads, (int64_t)128), 128, 0, st>>>(
        st_hi, st_lo, inc_hi, inc_lo, w.npos, w.len, w.val, w.fail);
    SKP_LAUNCHED(zig_attempt_kernel);
    zig_walk_kernel<<<(unsigned)w.nunits, kZE, 0, st>>>(w.len, w.nunits, w.exitmap, w.cnt);
    SKP_LAUNCHED(zig_walk_kernel);
    zig_group_kernel<<<(unsigned)cdiv(w.ngroups, (int64_t)4), 128, 0, st>>>(
        w.exitmap, w.cnt, w.nunits, w.gexit, w.gcnt);
    SKP_LAUNCHED(zig_group_kernel);
    zig_scan_groups_kernel<<<1, 32, 0, st>>>(w.gexit, w.gcnt, w.ngroups, count, w.gentry,
                                             w.goff, w.fail);
    SKP_LAUNCHED(zig_scan_groups_kernel);
    zig_units_kernel<<<(unsigned)cdiv(w.ngroups, (int64_t)128), 128, 0, st>>>(
        w.exitmap, w.cnt, w.nunits, w.ngroups, w.gentry, w.goff, w.uentry, w.uoff);
    SKP_LAUNCHED(zig_units_kernel);
    zig_write_kernel<T><<<(unsigned)w.nunits, 256, 0, st>>>(
        w.len, w.val, w.nunits, w.uentry, w.uoff, rows, cols, divisor, out, ldo, w.fail);
    SKP_LAUNCHED(zig_write_kernel);
    zig_report_kernel<<<1, 1, 0, st>>>(w.fail, fail_counter);
    SKP_LAUNCHED(zig_report_kernel);
    return SKP_OK;
}

}  // namespace
}  // namespace skp

using namespace skp;

extern "C" int64_t skp_gaussian_ws_bytes(int64_t count) {
    return count > 0 ? zig_layout(count, nullptr).bytes : 0;
}
extern "C" int skp_gaussian_f32(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                                int64_t rows, int64_t cols, double divisor, float* out,
                                int64_t ldo, int64_t* fail_counter, void* ws, int64_t ws_bytes,
                                void* stream) {
    return gaussian<float>(st_hi, st_lo, inc_hi, inc_lo, rows, cols, divisor, out, ldo,
                           fail_counter, ws, ws_bytes, SKP_STREAM(stream));
}
extern "C" int skp_gaussian_f64(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                                int64_t rows, int64_t cols, double divisor, double* out,
                                int64_t ldo, int64_t* fail_counter, void* ws, int64_t ws_bytes,
                                void* stream) {
    return gaussian<double>(st_hi, st_lo, inc_hi, inc_lo, rows, cols, divisor, out, ldo,
                            fail_counter, ws, ws_bytes, SKP_STREAM(stream));
}
