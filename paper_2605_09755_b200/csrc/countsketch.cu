// K1: on-device CountSketch generator, bit-exact with the reference draw
// (sketching.py:141-150 on numpy 2.3.5 PCG64), plus the CSC builder.
//
// PCG64 is an LCG on 128-bit state: x' = M x + inc.  k steps compose to
// x_k = M^k x + inc * G_k with G_k = sum_{i<k} M^i, so any draw position is
// one 128-bit multiply-add away from any other once (M^k, inc*G_k) is known.
// Keys kernel: one warp per row j; lane t walks draw positions j*r + t,
// t+32, ... with the stride-32 jump, keeps a register top-s list of
// (key = u64 >> 11, column), then the warp merges the 32 lists s times by
// (key, column) argmin -> ascending-key column order (== argpartition's
// prefix order on numpy 2.3.5, pinned by tests/golden).
// Signs kernel: draws n*r ... as 32-bit halves (low first), bit 31 -> +1.
#include "common.cuh"
#include "pcg.cuh"

namespace skp {
namespace {

constexpr int kWarps = 8;  // rows in flight per CTA

template <int SMAX>
__global__ void __launch_bounds__(kWarps * 32)
cs_keys_kernel(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t r,
               int s, int64_t j0, int64_t j1, int32_t* __restrict__ cols) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    const int64_t rows = j1 - j0;
    // contiguous row range per warp: row starts chain by one x -> step^r(x)
    const int64_t per = cdiv(rows, nwarps);
    int64_t jb = j0 + warp * per;
    int64_t je = jb + per < j1 ? jb + per : j1;
    if (jb >= je) return;
    const u128 inc = mk128(inc_hi, inc_lo);
    const Affine step_r = affine(jpow((uint64_t)r), inc);
    const Affine step_32 = affine(jpow(32), inc);
    // lane state at draw position jb*r + lane (state after jb*r + lane + 1 steps)
    u128 x = apply(affine(jpow((uint64_t)jb * (uint64_t)r + (uint64_t)lane + 1), inc),
                   mk128(st_hi, st_lo));
    for (int64_t j = jb; j < je; ++j) {
        uint64_t best[SMAX];
        int bidx[SMAX];
#pragma unroll
        for (int i = 0; i < SMAX; ++i) {
            best[i] = (i < s) ? ~0ULL : 0ULL;  // slots >= s never accept
            bidx[i] = 0x7fffffff;
        }
        uint64_t thr = ~0ULL;
        u128 y = x;
        for (int64_t c = lane; c < r; c += 32) {
            uint64_t key = xsl_rr(y) >> 11;
            y = apply(step_32, y);
            if (key < thr) {
                uint64_t k = key;
                int ci = (int)c;
#pragma unroll
                for (int i = 0; i < SMAX; ++i) {
                    if (k < best[i]) {
                        uint64_t tk = best[i]; best[i] = k; k = tk;
                        int tc = bidx[i]; bidx[i] = ci; ci = tc;
                    }
                }
#pragma unroll
                for (int i = 0; i < SMAX; ++i)
                    if (i == s - 1) thr = best[i];
            }
        }
        // warp merge: s rounds of (key, col) argmin over list heads
        int32_t* out = cols + (j - j0) * s;
        for (int t = 0; t < s; ++t) {
            uint64_t hk = best[0];
            int hc = bidx[0];
            uint64_t mk = hk;
            int mc = hc;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                uint64_t ok = __shfl_xor_sync(0xffffffffu, mk, o);
                int oc = __shfl_xor_sync(0xffffffffu, mc, o);
                if (ok < mk || (ok == mk && oc < mc)) { mk = ok; mc = oc; }
            }
            if (lane == 0) out[t] = mc;
            if (hk == mk && hc == mc) {  // winner pops its head
#pragma unroll
                for (int i = 0; i < SMAX - 1; ++i) { best[i] = best[i + 1]; bidx[i] = bidx[i + 1]; }
                best[SMAX - 1] = ~0ULL;
                bidx[SMAX - 1] = 0x7fffffff;
            }
        }
        x = apply(step_r, x);
    }
}

// Signs: element e = j*s + t is 32-bit value u0 + e of the generator's uint32
// stream (value h = half h&1 of 64-bit draw h>>1, low half first); bit 31 set
// -> +1 (Lemire with range 2 never rejects).  u0 = the uint32 values the
// column phase consumed: numpy's PCG64 keeps the unused high half of a draw in
// the bit generator (has_uint32) across integers() calls, so after an odd
// number of Lemire-32 column draws (s == 1) the first sign is that buffered
// high half.  Each thread owns kSignDraws consecutive 64-bit draws.
constexpr int kSignDraws = 16;

__global__ void cs_signs_kernel(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                                const int64_t* __restrict__ u0_dev, uint64_t u0_host, int64_t e0,
                                int64_t e1, int8_t* __restrict__ signs) {
    const u128 inc = mk128(inc_hi, inc_lo);
    const int64_t u0 = u0_dev ? *u0_dev : (int64_t)u0_host;
    // first and last draw covering elements [e0, e1)
    const int64_t dfirst = (u0 + e0) >> 1, dlast = (u0 + e1 - 1) >> 1;
    int64_t d = dfirst + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kSignDraws;
    if (d > dlast) return;
    u128 x = apply(affine(jpow((uint64_t)d + 1), inc), mk128(st_hi, st_lo));
    const Affine one{pcg_mult(), inc};
    for (int k = 0; k < kSignDraws && d <= dlast; ++k, ++d) {
        uint64_t v = xsl_rr(x);
        x = apply(one, x);
        const int64_t e = 2 * d - u0;  // element of the low half
        if (e >= e0 && e < e1) signs[e - e0] = ((uint32_t)v >> 31) ? 1 : -1;
        if (e + 1 >= e0 && e + 1 < e1) signs[e + 1 - e0] = ((uint32_t)(v >> 32) >> 31) ? 1 : -1;
    }
}
// grid for cs_signs_kernel over elements [e0, e1) (any u0)
inline int sign_blocks(int64_t e0, int64_t e1) {
    const int64_t draws = (e1 - e0) / 2 + 2;
    return (int)cdiv(cdiv(draws, (int64_t)kSignDraws), (int64_t)256);
}

// ---- s == 1: cols = integers(0, r) by Lemire-32 with rejection --------------
// Candidate halves h = 0..H-1 (draw h/2, low half first).  Accepted halves in
// order give cols[0..n).  Three passes: per-tile accept counts, scan, write.
constexpr int kTile = 1024;  // halves per CTA tile (256 threads x 4)

__device__ __forceinline__ uint32_t half_at(u128 x_after_draw, int which) {
    uint64_t v = xsl_rr(x_after_draw);
    return which ? (uint32_t)(v >> 32) : (uint32_t)v;
}

__global__ void s1_count_kernel(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                                int64_t H, uint32_t excl, uint32_t thr, int32_t* tile_cnt) {
    __shared__ int scratch[32];
    const u128 inc = mk128(inc_hi, inc_lo);
    int64_t h0 = (int64_t)blockIdx.x * kTile + threadIdx.x * 4;  // 4 halves = 2 draws
    int cnt = 0;
    if (h0 < H) {
        u128 x = apply(affine(jpow((uint64_t)(h0 >> 1) + 1), inc), mk128(st_hi, st_lo));
        const Affine one{pcg_mult(), inc};
        for (int k = 0; k < 4; ++k) {
            int64_t h = h0 + k;
            if (h >= H) break;
            if (k == 2) x = apply(one, x);
            uint32_t u = half_at(x, (int)(h & 1));
            uint32_t left = (uint32_t)((uint64_t)u * excl);
            cnt += !(left < thr);
        }
    }
    int tot = block_sum<int>(cnt, scratch);
    if (threadIdx.x == 0) tile_cnt[blockIdx.x] = tot;
}

__global__ void s1_scan_kernel(int32_t* tile_cnt, int64_t ntiles, int64_t* total) {
    // single CTA exclusive scan (ntiles is small: H / 1024)
    __shared__ int64_t carry;
    __shared__ int64_t buf[1024];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < ntiles; base += 1024) {
        int64_t i = base + threadIdx.x;
        int64_t v = i < ntiles ? tile_cnt[i] : 0;
        buf[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            int64_t t = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
            __syncthreads();
            buf[threadIdx.x] += t;
            __syncthreads();
        }
        if (i < ntiles) tile_cnt[i] = (int32_t)(carry + buf[threadIdx.x] - v);
        __syncthreads();
        if (threadIdx.x == 1023) carry += buf[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void s1_write_kernel(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                                int64_t H, uint32_t excl, uint32_t thr, const int32_t* tile_off,
                                int64_t n, int64_t j0, int64_t j1, int32_t* cols,
                                int64_t* sign_d0) {
    __shared__ int warp_tot[8];
    const u128 inc = mk128(inc_hi, inc_lo);
    int64_t h0 = (int64_t)blockIdx.x * kTile + threadIdx.x * 4;
    uint32_t val[4];
    bool acc[4];
    int cnt = 0;
    if (h0 < H) {
        u128 x = apply(affine(jpow((uint64_t)(h0 >> 1) + 1), inc), mk128(st_hi, st_lo));
        const Affine one{pcg_mult(), inc};
        for (int k = 0; k < 4; ++k) {
            int64_t h = h0 + k;
            acc[k] = false;
            if (h >= H) continue;
            if (k == 2) x = apply(one, x);
            uint32_t u = half_at(x, (int)(h & 1));
            uint64_t mm = (uint64_t)u * excl;
            acc[k] = !((uint32_t)mm < thr);
            val[k] = (uint32_t)(mm >> 32);
            cnt += acc[k];
        }
    } else {
        for (int k = 0; k < 4; ++k) acc[k] = false;
    }
    // block exclusive scan of cnt (256 threads)
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    int woff = 0;
    for (int i = 0; i < w; ++i) woff += warp_tot[i];
    int64_t rank = (int64_t)tile_off[blockIdx.x] + woff + incl - cnt;
    for (int k = 0; k < 4; ++k) {
        if (!acc[k]) continue;
        if (rank >= j0 && rank < j1) cols[rank - j0] = (int32_t)val[k];
        if (rank == n - 1) {
            int64_t halves_used = h0 + k + 1;
            *sign_d0 = halves_used;  // uint32 values consumed: the signs continue from here
        }
        ++rank;
    }
}

}  // namespace
}  // namespace skp

using namespace skp;

extern "C" int64_t skp_countsketch_ws_bytes(int64_t n, int64_t r, int32_t s) {
    (void)r;
    if (s != 1) return 0;
    int64_t H = n + n / 64 + 4096;
    int64_t ntiles = cdiv(H, kTile);
    return 64 + ntiles * 4 + 64;
}

extern "C" int skp_countsketch_gen(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi,
                                   uint64_t inc_lo, int64_t n, int64_t r, int32_t s, int64_t j0,
                                   int64_t j1, int32_t* cols, int8_t* signs, void* ws,
                                   int64_t ws_bytes, void* stream) {
    SKP_ARG(n >= 1 && r >= 1, "countsketch needs n >= 1 and r >= 1, got n=%lld r=%lld",
            (long long)n, (long long)r);
    SKP_ARG(s >= 1 && s <= r, "countsketch needs 1 <= s <= r, got s=%d, r=%lld", s, (long long)r);
    SKP_ARG(0 <= j0 && j0 <= j1 && j1 <= n, "bad row range [%lld, %lld)", (long long)j0,
            (long long)j1);
    if (s > 32) {
        set_error("unsupported: device countsketch supports s <= 32 (got s=%d)", s);
        return SKP_ERR_UNSUPPORTED;
    }
    if (r > 0x7fffffffLL) {
        set_error("unsupported: device countsketch supports r < 2^31 (got r=%lld)", (long long)r);
        return SKP_ERR_UNSUPPORTED;
    }
    if (j0 == j1) return SKP_OK;
    cudaStream_t st = SKP_STREAM(stream);
    if (s == 1) {
        SKP_ARG(ws != nullptr && ws_bytes >= skp_countsketch_ws_bytes(n, r, s),
                "countsketch s=1 needs %lld bytes of workspace",
                (long long)skp_countsketch_ws_bytes(n, r, s));
        int64_t* d_total = reinterpret_cast<int64_t*>(ws);
        int64_t* d_sign0 = d_total + 1;
        int32_t* tiles = reinterpret_cast<int32_t*>(d_total + 8);
        if (r == 1) {
            // rng == 0: all zeros, no draws consumed (numpy random_bounded_uint64_fill)
            SKP_CUDA(cudaMemsetAsync(cols, 0, sizeof(int32_t) * (j1 - j0), st));
            cs_signs_kernel<<<sign_blocks(j0, j1), 256, 0, st>>>(st_hi, st_lo, inc_hi, inc_lo,
                                                                 nullptr, 0, j0, j1, signs);
            SKP_LAUNCHED(cs_signs_kernel);
            return SKP_OK;
        }
        const uint32_t excl = (uint32_t)r;  // rng + 1
        const uint32_t thr = (uint32_t)(0u - excl) % excl;
        int64_t H = n + n / 64 + 4096;  // candidate halves; expected rejections << n/64
        int64_t ntiles = cdiv(H, kTile);
        s1_count_kernel<<<(int)ntiles, 256, 0, st>>>(st_hi, st_lo, inc_hi, inc_lo, H, excl, thr,
                                                    tiles);
        SKP_LAUNCHED(s1_count_kernel);
        s1_scan_kernel<<<1, 1024, 0, st>>>(tiles, ntiles, d_total);
        SKP_LAUNCHED(s1_scan_kernel);
        int64_t total = 0;
        SKP_CUDA(cudaMemcpyAsync(&total, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SKP_CUDA(cudaStreamSynchronize(st));
        if (total < n) {
            set_error("unsupported: Lemire rejection rate too high for r=%lld (accepted %lld of "
                      "%lld)", (long long)r, (long long)total, (long long)H);
            return SKP_ERR_UNSUPPORTED;
        }
        s1_write_kernel<<<(int)ntiles, 256, 0, st>>>(st_hi, st_lo, inc_hi, inc_lo, H, excl, thr,
                                                    tiles, n, j0, j1, cols, d_sign0);
        SKP_LAUNCHED(s1_write_kernel);
        cs_signs_kernel<<<sign_blocks(j0, j1), 256, 0, st>>>(st_hi, st_lo, inc_hi, inc_lo, d_sign0,
                                                             0, j0, j1, signs);
        SKP_LAUNCHED(cs_signs_kernel);
        return SKP_OK;
    }
    int dev = 0, sms = 148;
    SKP_CUDA(cudaGetDevice(&dev));
    SKP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int64_t rows = j1 - j0;
    // enough warps to fill the machine, >= 4 rows per warp when possible
    int64_t want = cdiv(rows, 4);
    int64_t blocks = cdiv(want, kWarps);
    int64_t maxb = (int64_t)sms * 16;
    if (blocks > maxb) blocks = maxb;
    if (blocks < 1) blocks = 1;
    if (s <= 8)
        cs_keys_kernel<8><<<(int)blocks, kWarps * 32, 0, st>>>(st_hi, st_lo, inc_hi, inc_lo, r, s,
                                                             j0, j1, cols);
    else
        cs_keys_kernel<32><<<(int)blocks, kWarps * 32, 0, st>>>(st_hi, st_lo, inc_hi, inc_lo, r,
                                                              s, j0, j1, cols);
    SKP_LAUNCHED(cs_keys_kernel);
    // the key phase consumed n*r 64-bit draws (2*n*r uint32 values, none buffered)
    int64_t e0 = j0 * s, e1 = j1 * s;
    cs_signs_kernel<<<sign_blocks(e0, e1), 256, 0, st>>>(st_hi, st_lo, inc_hi, inc_lo, nullptr,
                                                         2 * (uint64_t)n * (uint64_t)r, e0, e1,
                                                         signs);
    SKP_LAUNCHED(cs_signs_kernel);
    return SKP_OK;
}

// ------------------------------------------------------------------ CSC ---
namespace skp {
namespace {

__global__ void csc_count_kernel(const int32_t* __restrict__ cols, int64_t nnz,
                                 int32_t* __restrict__ cnt) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[cols[e]], 1);
}

__global__ void csc_scan_kernel(const int32_t* __restrict__ cnt, int64_t r,
                                int32_t* __restrict__ colptr) {
    __shared__ int64_t buf[1024];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < r; base += 1024) {
        int64_t i = base + threadIdx.x;
        int64_t v = i < r ? cnt[i] : 0;
        buf[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            int64_t t = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
            __syncthreads();
            buf[threadIdx.x] += t;
            __syncthreads();
        }
        if (i < r) colptr[i] = (int32_t)(carry + buf[threadIdx.x] - v);
        __syncthreads();
        if (threadIdx.x == 1023) carry += buf[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) colptr[r] = (int32_t)carry;
}

__global__ void csc_fill_kernel(const int32_t* __restrict__ cols, const int8_t* __restrict__ signs,
                                int64_t nnz, int s, const int32_t* __restrict__ colptr,
                                int32_t* __restrict__ cursor, int32_t* __restrict__ entries) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        int c = cols[e];
        int pos = atomicAdd(&cursor[c], 1);
        uint32_t j = (uint32_t)(e / s);
        entries[colptr[c] + pos] = (int32_t)(j | (signs[e] < 0 ? 0x80000000u : 0u));
    }
}

// deterministic order: sort each column's entries by row index j
__global__ void csc_sort_kernel(const int32_t* __restrict__ colptr, int64_t r,
                                int32_t* __restrict__ entries) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < r;
         c += (int64_t)gridDim.x * blockDim.x) {
        int b = colptr[c], e = colptr[c + 1];
        for (int i = b + 1; i < e; ++i) {
            uint32_t v = (uint32_t)entries[i];
            uint32_t key = v & 0x7fffffffu;
            int k = i - 1;
            while (k >= b && ((uint32_t)entries[k] & 0x7fffffffu) > key) {
                entries[k + 1] = entries[k];
                --k;
            }
            entries[k + 1] = (int32_t)v;
        }
    }
}

}  // namespace
}  // namespace skp

extern "C" int64_t skp_countsketch_csc_ws_bytes(int64_t n, int32_t s, int64_t r) {
    (void)n;
    (void)s;
    return 2 * (r + 1) * (int64_t)sizeof(int32_t) + 256;
}

extern "C" int skp_countsketch_csc(const int32_t* cols, const int8_t* signs, int64_t n, int32_t s,
                                   int64_t r, int32_t* colptr, int32_t* entries, void* ws,
                                   int64_t ws_bytes, void* stream) {
    SKP_ARG(n >= 1 && s >= 1 && r >= 1, "bad csc sizes");
    SKP_ARG(n * (int64_t)s < 0x7fffffffLL, "csc: n*s must be < 2^31");
    SKP_ARG(ws != nullptr && ws_bytes >= skp_countsketch_csc_ws_bytes(n, s, r),
            "csc needs %lld bytes of workspace", (long long)skp_countsketch_csc_ws_bytes(n, s, r));
    cudaStream_t st = SKP_STREAM(stream);
    int32_t* cnt = reinterpret_cast<int32_t*>(ws);
    int32_t* cursor = cnt + (r + 1);
    SKP_CUDA(cudaMemsetAsync(ws, 0, 2 * (r + 1) * sizeof(int32_t), st));
    int64_t nnz = n * s;
    int blocks = (int)(cdiv(nnz, 256) < 4096 ? cdiv(nnz, 256) : 4096);
    csc_count_kernel<<<blocks, 256, 0, st>>>(cols, nnz, cnt);
    SKP_LAUNCHED(csc_count_kernel);
    csc_scan_kernel<<<1, 1024, 0, st>>>(cnt, r, colptr);
    SKP_LAUNCHED(csc_scan_kernel);
    csc_fill_kernel<<<blocks, 256, 0, st>>>(cols, signs, nnz, s, colptr, cursor, entries);
    SKP_LAUNCHED(csc_fill_kernel);
    int sb = (int)(cdiv(r, 128) < 4096 ? cdiv(r, 128) : 4096);
    csc_sort_kernel<<<sb, 128, 0, st>>>(colptr, r, entries);
    SKP_LAUNCHED(csc_sort_kernel);
    return SKP_OK;
}
