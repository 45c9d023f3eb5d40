// K2 v2 (fp32): A~ = A . S as a ROW GATHER with a register-resident,
// bank-conflict-free schedule.
//
// Output column c of A~ is  sum_e sign_e * A[:, j_e]  over the ~n*s/l (C3:
// 33) CountSketch entries of column c.  Lane = output column: each thread keeps
// its column's entries in registers as smem byte addresses (bit 31 = negate),
// and every row of A is streamed whole into a double-buffered shared-memory
// row by 1-D bulk copies.  One step = 4 instructions for the warp's 32 columns:
//     LOP3 (address) -> LDS -> LOP3 (sign xor) -> FADD
// No per-(chunk, column) metadata, no padding slots, no transposes, and the
// warp's 32 results of a row are one coalesced 128-byte store.
//
// Bank conflicts: the 32 lanes of a warp load 32 data-dependent words of the
// row; the order of each lane's entries is scheduled offline (per sketch, on
// the device) so that at every step the warp touches 32 distinct banks -- an
// edge colouring of the lane x bank multigraph (plan 2) in as many steps as
// the busiest lane has entries; a bank with more entries than that meets
// itself in a few steps (2-way conflicts).  Lanes without an entry at a step
// read a zero word in a free bank.  Columns are sorted by entry count inside
// each slice, so the 32 lanes of a warp carry about the same number of
// entries.  The sort permutes the OUTPUT COLUMNS: the kernel
// writes A~ P, and the range finder multiplies by P^T Omega instead of Omega
// (Y = A~ Omega = (A~ P)(P^T Omega)); apply_right keeps K2 v1's column order.
//
// CTA = one slice of <= kGCols = 896 output columns (28 warps; the slices are
// balanced to gather_width columns each); the last warp to finish a row
// refills its buffer (bulk copy of the row two ahead).  Grid = G row groups x
// P slices.  The CTAs of a row group read the same rows but drift apart, so
// ~3x |A| comes from HBM (ncu, C3: 50 GB).  Pacing them to within L2 reach (a
// group row counter, tested) cut that to 17.2 GB but cost 12-25% time: the
// kernel is bound by its shared-memory gathers, not by HBM.
//
// Non-finite test: every column of A feeds s >= 1 nonzero (+-1/sqrt(s))
// entries, so A has a non-finite entry iff A~ does -- each thread tests the
// value it stores (one instruction per row; a fused fp64 ||A||^2 here cost 20%
// of the kernel).  ||A||_F^2, when asked for, is a separate HBM-bound pass
// (skp_sumsq).
#include <cuda.h>

#include <algorithm>
#include <stdlib.h>
#include <type_traits>

#include "common.cuh"

extern "C" int skp_sumsq_f32(const float* X, int64_t rows, int64_t cols, int64_t ld, double* out,
                             int64_t* nonfinite, void* stream);  // sketch.cu

namespace skp {

namespace {

constexpr int kGW = 28;                   // compute warps per CTA
constexpr int kGCols = kGW * 32;          // output columns per slice
// no producer warp; 28 warps x 72 registers (7 warps per SMSP: 16128 <=
// 16384 registers) so that C3's l = 4000 takes 5 slices of 800 columns instead
// of 6 of 672 -- each row is bulk-copied into one CTA fewer -- with 96 spare
// lanes per slice for splitting the heavy columns.  44 register-resident
// steps cover C3's heaviest warp (44); the last warp to finish a row issues
// the bulk copy of the row NB ahead
constexpr int kGThreads = 32 * kGW;
constexpr int kGTReg = 44;                // schedule steps held in registers
constexpr int kGTMax = 128;               // schedule steps per warp (the rest: L1/global)
constexpr unsigned long long kGPlanFailMark = 1ull << 40;  // added to *nonfinite
constexpr int kGBufWords = 24608;         // row buffer: n <= 24576 floats + 32 zero words
constexpr uint32_t kGBufBytes = kGBufWords * 4;  // 98432, a multiple of 128
// three row buffers (NB = 3, rows <= 75 KB; tested, not launched): warps of a CTA may
// drift two rows apart before the slowest gates a refill.  Measured at C3:
// 11.54 -> 11.46 ms with 6 slices of 24 warps, but 9.86 (two) vs 10.01 ms
// (three) with 5 slices of 28 warps, and ~20% more DRAM re-reads -- so two
// buffers are the default
constexpr uint32_t kGBufBytes3 = 75776;  // 18944 words, a multiple of 128
constexpr int kGN3 = kGBufBytes3 / 4 - 64;
template <int NB>
struct GBuf {
    static constexpr uint32_t bytes = NB == 2 ? kGBufBytes : kGBufBytes3;
    static constexpr size_t smem = NB * (size_t)bytes + 64;
};

__device__ __forceinline__ uint32_t g_smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void g_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(g_smem_u32(bar)), "r"(count));
}
// try_wait with a suspend-time hint: a warp whose row has not landed sleeps in
// the barrier unit until the phase completes (or ~1 ms) instead of spinning.
// The spin form issued ~13 polls per row, each with the watchdog's clock
// arithmetic if-converted into it: 37% of K2's instructions at C5 in an
// issue-bound kernel (profiles/r02za_c5_pair_full.txt, before this change).
__device__ __forceinline__ bool g_mbar_try(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity), "n"(1000000)
        : "memory");
    return ok != 0;
}
// (a = the barrier's shared address)
__device__ __forceinline__ void g_mbar_wait_a(uint32_t a, uint32_t parity) {
    if (g_mbar_try(a, parity)) return;
    const long long t0 = clock64();
    while (!g_mbar_try(a, parity))
        if (clock64() - t0 > (long long)40e9) __trap();
}
__device__ __forceinline__ void g_mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = g_smem_u32(bar);
    if (g_mbar_try(a, parity)) return;
    // watchdog (cold): a protocol bug becomes a trap (error), never a hung GPU
    const long long t0 = clock64();
    while (!g_mbar_try(a, parity))
        if (clock64() - t0 > (long long)40e9) __trap();
}
__device__ __forceinline__ void g_mbar_arrive_e(uint64_t* bar) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
                 "@p mbarrier.arrive.shared::cta.b64 _, [%0];\n\t}" ::"r"(g_smem_u32(bar))
                 : "memory");
}
// elected lane: expect `bytes` on bar, then bulk-copy them global -> smem
__device__ __forceinline__ void g_bulk_load_e(uint32_t dst, const void* src, uint32_t bytes,
                                              uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n\t"
        "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %3, "
        "[%2];\n\t}" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(g_smem_u32(bar)), "r"(bytes)
        : "memory");
}

// ---- plan 1: per-slice lane table ---------------------------------------------
// Slice p owns output positions [p*width, p*width + nc_p) (width = the balanced
// slice width, gather_width).  A warp's schedule is as long as its heaviest
// lane, and columns sorted by entry count leave the heavy warps ~1.5x longer
// than the mean (C3: 52-56 steps vs 35 -- warps idle a third of the time).
// So columns with more than `cap` entries are split into two half-columns on
// an adjacent lane pair (2k, 2k+1) whose sums the kernel combines with one
// shuffle; cap is the smallest value >= the mean count for which the lanes
// still fit the CTA's 32*kGW.  Lane units (1 or 2 lanes) are sorted by
// per-lane count, descending, and placed in order (a pair never straddles an
// even lane boundary; the hole it skips is filled by the next single).
// Per lane: seg_beg / seg_cnt (its range of the column's CSC entries) and
// lanepos = output position | kGPrimary (add lane+1's sum), or -1 (no write).
// perm[pos] = the column written at position pos (compact: the first r
// entries), -1 for pos in [r, P*kGCols).  One block per slice.
constexpr int kGPrimary = 1 << 30;
constexpr int kGMaxPass = 4;  // column passes: n <= 4 x 24576
struct GSched {
    int H;
    uint32_t* sched[kGMaxPass];
    int32_t* tw[kGMaxPass];
};
__global__ void __launch_bounds__(256)
gather_sort_kernel(const int32_t* __restrict__ colptr, const int32_t* __restrict__ entries,
                   int64_t r, int width, int64_t slots, int H, int npass,
                   int32_t* __restrict__ perm, int32_t* __restrict__ seg_beg,
                   int32_t* __restrict__ seg_cnt, int32_t* __restrict__ lanepos,
                   int32_t* __restrict__ fail) {
    __shared__ int key[kGCols];        // column entry counts
    __shared__ int ucnt[kGCols];       // per-lane count of the column's unit
    __shared__ int order[kGCols];      // units in placement order (column index)
    __shared__ int lane_col[kGCols];   // lane -> column (-1 empty)
    __shared__ int lane_part[kGCols];  // 0 single, 1 first half (primary), 2 second half
    // entry counts over all column passes: a lane's per-pass count is ~1/H
    // of it, so totals up to H * kGTMax are schedulable
    constexpr int kHist = kGTMax * kGMaxPass + 2;
    __shared__ int hist[kHist];
    __shared__ int s_cap;
    // column passes (n > one row buffer): bnd[v][h] = first entry of column v
    // with j >= h * npass (entries are ascending in j)
    __shared__ int bnd[kGCols][kGMaxPass + 1];
    const int64_t c0 = (int64_t)blockIdx.x * width;
    const int nc = (int)(r - c0 < width ? r - c0 : width);
    const int lanes = kGCols;
    for (int v = threadIdx.x; v < kGCols; v += blockDim.x) {
        key[v] = v < nc ? colptr[c0 + v + 1] - colptr[c0 + v] : -1;
        lane_col[v] = -1;
        lane_part[v] = 0;
    }
    for (int v = threadIdx.x; v < kHist; v += blockDim.x) hist[v] = 0;
    const int cmax = H * kGTMax + 1;  // histogram clamp
    if (blockIdx.x == 0)
        for (int64_t v = r + threadIdx.x; v < slots; v += blockDim.x) perm[v] = -1;
    __syncthreads();
    for (int v = threadIdx.x; v < nc; v += blockDim.x) {
        atomicAdd(&hist[min(key[v], cmax)], 1);
        const int b0 = colptr[c0 + v], b1 = colptr[c0 + v + 1];
        bnd[v][0] = b0;
        bnd[v][H] = b1;
        for (int h = 1; h < H; ++h) {
            const int jt = h * npass;
            int lo = b0, hi = b1;  // first index with (entry & 0x7fffffff) >= jt
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if ((entries[mid] & 0x7fffffff) < jt) lo = mid + 1;
                else hi = mid;
            }
            bnd[v][h] = lo;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long tot = 0;
        for (int c = 0; c <= cmax; ++c) tot += (long long)c * hist[c];
        const int mean = nc ? (int)((tot + nc - 1) / nc) : 0;
        // columns above cap become 2 lanes (+ at most one hole each)
        int above = 0, cap = cmax;
        for (int c = cmax; c >= mean; --c) {
            if (nc + 2 * (above + hist[c]) > lanes) break;
            above += hist[c];
            cap = c - 1;
        }
        s_cap = max(cap, mean);
    }
    __syncthreads();
    const int cap = s_cap;
    for (int v = threadIdx.x; v < kGCols; v += blockDim.x) {
        int u = v < nc ? (key[v] > cap ? (key[v] + 1) / 2 : key[v]) : -1;
        // several column passes: a warp runs, in every pass, as many steps as
        // its heaviest lane has entries IN THAT PASS, so lanes are grouped by
        // their largest per-pass count, not by their total (C5, two passes of
        // ~16 entries per column: lanes of equal totals differ by +-3 per
        // pass and the warps ran 24.0 steps per pass for a mean of 16.4; now
        // 20.4 -- padding 1.58 -> 1.34, 2-way conflicts 1.07 -> 1.21 per LDS)
        if (v < nc && H > 1) {
            const int beg = bnd[v][0], cnt = key[v], half = (cnt + 1) / 2;
            const bool pair = cnt > cap;
            u = 0;
            for (int part = 0; part < (pair ? 2 : 1); ++part) {
                const int pb = part ? beg + half : beg;
                const int pe = pair && !part ? beg + half : beg + cnt;
                for (int h = 0; h < H; ++h)
                    u = max(u, min(pe, bnd[v][h + 1]) - max(pb, bnd[v][h]));
            }
        }
        ucnt[v] = u;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < nc; v += blockDim.x) {
        const int kv = ucnt[v];
        int rank = 0;
        for (int u = 0; u < nc; ++u) {
            const int ku = ucnt[u];
            rank += (ku > kv) || (ku == kv && u < v);
        }
        order[rank] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int pos = 0, hole = -1;
        for (int k = 0; k < nc; ++k) {
            const int v = order[k];
            const bool pair = key[v] > cap;
            if (pair ? pos + 2 + (pos & 1) > lanes : (hole < 0 && pos >= lanes)) {
                atomicOr(fail, 1);  // lanes exhausted (mean count near kGTMax): no plan
                break;
            }
            if (pair) {
                if (pos & 1) {  // keep the pair on (2k, 2k+1): skip a lane
                    if (hole < 0) hole = pos;
                    ++pos;
                }
                lane_col[pos] = v;
                lane_part[pos] = 1;
                lane_col[pos + 1] = v;
                lane_part[pos + 1] = 2;
                pos += 2;
            } else if (hole >= 0) {
                lane_col[hole] = v;
                hole = -1;
            } else {
                lane_col[pos++] = v;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // output positions in lane order
        int k = 0;
        for (int l = 0; l < lanes; ++l) {
            const int v = lane_col[l];
            const int64_t g = (int64_t)blockIdx.x * kGCols + l;
            const int64_t pstride = slots;  // per-pass table stride (P * kGCols)
            if (v < 0) {
                for (int h = 0; h < H; ++h) {
                    seg_beg[h * pstride + g] = 0;
                    seg_cnt[h * pstride + g] = 0;
                }
                lanepos[g] = -1;
                continue;
            }
            const int beg = colptr[c0 + v], cnt = key[v];
            const int half = (cnt + 1) / 2;
            // this lane's part of the column, intersected with each pass's j range
            const int pb = lane_part[l] == 2 ? beg + half : beg;
            const int pe = lane_part[l] == 1 ? beg + half : beg + cnt;
            for (int h = 0; h < H; ++h) {
                const int sb = max(pb, bnd[v][h]), se = min(pe, bnd[v][h + 1]);
                seg_beg[h * pstride + g] = sb;
                seg_cnt[h * pstride + g] = max(0, se - sb);
            }
            if (lane_part[l] == 2) {
                lanepos[g] = -1;
            } else {
                perm[c0 + k] = (int32_t)(c0 + v);
                lanepos[g] = (int32_t)(c0 + k) | (lane_part[l] == 1 ? kGPrimary : 0);
                ++k;
            }
        }
    }
}

// ---- plan 2: step schedule, one block per warp schedule ----------------------
// sched[(wg*kGTMax + t)*32 + lane] = byte offset into the row buffer (bit 31:
// negate); tw[wg] = steps (a multiple of 4); fail |= 1 when a warp needs more
// than kGTMax steps (the caller then keeps K2 v1).
// The warp's entries are the edges of a bipartite multigraph lanes x banks
// (bank = column index mod 32); a step is a set of edges with each lane at most
// once, and its shared-memory wavefronts are the most lanes on one bank.  The
// warp must take L = (most entries on one lane) steps; a bank with more than L
// entries is split into virtual banks of <= L entries each, and the graph
// lanes x virtual banks is coloured with exactly L colours (Koenig's theorem):
// L steps, and a 2-way conflict only where both halves of an overloaded bank
// meet in one step (C3: ~1.1 wavefronts per LDS; a greedy colouring measured
// 2.47, and a conflict-free colouring needs max(L, bank degree) steps -- 30%
// more, and slower).
// Colouring (one thread; ~1000 edges per warp): an edge takes a colour free at
// both ends; otherwise, with a free at its lane and b free at its bank, the
// a/b alternating path from the bank is swapped first (it cannot reach the
// lane: bipartite), which frees a at the bank.  Lanes idle at a step read a
// zero word in a distinct unused bank.
constexpr int kGCW = kGTMax / 32;  // colour mask words
constexpr int kGVB = 4;            // virtual banks per bank
__device__ __forceinline__ int g_first_free(const uint32_t* m0, const uint32_t* m1, int lim) {
#pragma unroll
    for (int w = 0; w < kGCW; ++w) {
        const uint32_t f = ~(m0[w] | (m1 ? m1[w] : 0u));
        if (f) {
            const int c = w * 32 + __ffs(f) - 1;
            return c < lim ? c : -1;
        }
    }
    return -1;
}
__global__ void __launch_bounds__(32)
gather_sched_kernel(const int32_t* __restrict__ seg_beg, const int32_t* __restrict__ seg_cnt,
                    const int32_t* __restrict__ entries, int nwarps, int64_t n, int npass,
                    GSched ps, int32_t* __restrict__ fail) {
    __shared__ uint8_t lane_bank[32][kGTMax];        // virtual bank of lane at colour c (0xff: none)
    __shared__ uint8_t bank_lane[32 * kGVB][kGTMax];  // lane on virtual bank at colour c
    __shared__ uint32_t val[32][kGTMax];              // the entry at (lane, colour)
    __shared__ uint32_t lmask[32][kGCW], bmask[32 * kGVB][kGCW];  // colours in use
    __shared__ int bdeg[32], bfill[32], sbeg[32], scnt[32];
    const int lane = threadIdx.x;
    const int h = blockIdx.x / nwarps, wg = blockIdx.x % nwarps;  // column pass, warp
    const uint32_t j0 = (uint32_t)(h * npass);
    const int64_t nh = std::min<int64_t>(npass, n - j0);
    uint32_t* sched = ps.sched[h];
    int32_t* tw = ps.tw[h];
    const uint32_t zero_word = (uint32_t)((nh + 31) / 32 * 32);  // 32 zero words after the row
    const int64_t ti = (int64_t)h * nwarps * 32 + (int64_t)wg * 32 + lane;
    const int beg = seg_beg[ti];  // this lane's (half-)column, this pass's j range
    const int cnt = seg_cnt[ti];
    sbeg[lane] = beg;
    scnt[lane] = cnt;
    bdeg[lane] = bfill[lane] = 0;
    for (int c = 0; c < kGTMax; ++c) {
        lane_bank[lane][c] = 0xff;
#pragma unroll
        for (int k = 0; k < kGVB; ++k) bank_lane[lane + 32 * k][c] = 0xff;
    }
#pragma unroll
    for (int w = 0; w < kGCW; ++w) {
        lmask[lane][w] = 0u;
#pragma unroll
        for (int k = 0; k < kGVB; ++k) bmask[lane + 32 * k][w] = 0u;
    }
    __syncwarp();
    for (int k = 0; k < cnt; ++k) atomicAdd(&bdeg[(uint32_t)entries[beg + k] & 31u], 1);
    __syncwarp();
    int L = cnt, B = bdeg[lane];
    for (int o = 16; o; o >>= 1) {
        L = max(L, __shfl_xor_sync(0xffffffffu, L, o));
        B = max(B, __shfl_xor_sync(0xffffffffu, B, o));
    }
    const int T = (L + 3) & ~3;
    // the kernel runs T steps (a multiple of 4) anyway: the colouring gets all
    // T colours, so banks with up to T entries need no conflict at all
    // (C3: 1.60 -> 1.46 wavefronts per LDS, K2 10.0 -> 9.7 ms)
    const int C = T;
    if (T > kGTMax || B > kGVB * C) {
        if (lane == 0) {
            atomicOr(fail, 1);
            tw[wg] = 0;
        }
        return;
    }
    if (lane == 0) {
        auto put = [&](int l, int b, int c, uint32_t v) {
            lane_bank[l][c] = (uint8_t)b;
            bank_lane[b][c] = (uint8_t)l;
            val[l][c] = v;
            lmask[l][c >> 5] |= 1u << (c & 31);
            bmask[b][c >> 5] |= 1u << (c & 31);
        };
        auto drop = [&](int l, int b, int c) {
            lane_bank[l][c] = 0xff;
            bank_lane[b][c] = 0xff;
            lmask[l][c >> 5] &= ~(1u << (c & 31));
            bmask[b][c >> 5] &= ~(1u << (c & 31));
        };
        // (lane, vbank, colour) of the alternating path: each lane at most once
        uint32_t path[2 * 32], pv[2 * 32];
        // the overflow edges of overloaded banks first: they take the lowest
        // colours, so their 2-way conflicts gather in few steps
        for (int pass = 0; pass < 2; ++pass) {
          for (int q = 0; q < 32; ++q) bfill[q] = 0;
          for (int u = 0; u < 32; ++u) {
            for (int k = 0; k < scnt[u]; ++k) {
                const uint32_t v = (uint32_t)entries[sbeg[u] + k];
                const int rb = (int)(v & 31u);
                const int vi = bfill[rb]++;  // this edge's index on its bank
                if ((vi >= C) != (pass == 0)) continue;
                const int b = rb + 32 * (vi / C);  // virtual bank (<= C entries each)
                int c = g_first_free(lmask[u], bmask[b], C);
                if (c < 0) {
                    const int ca = g_first_free(lmask[u], nullptr, C);  // free at the lane
                    const int cb = g_first_free(bmask[b], nullptr, C);  // free at the bank
                    // swap colours ca <-> cb on the path bank b -ca- lane -cb- bank ...
                    int np = 0, x = b;
                    for (;;) {
                        const int l = bank_lane[x][ca];
                        if (l == 0xff) break;
                        path[np++] = (uint32_t)l | ((uint32_t)x << 8) | ((uint32_t)ca << 16);
                        const int y = lane_bank[l][cb];
                        if (y == 0xff) break;
                        path[np++] = (uint32_t)l | ((uint32_t)y << 8) | ((uint32_t)cb << 16);
                        x = y;
                    }
                    for (int q = 0; q < np; ++q) {
                        const int l = path[q] & 0xff, bb = (path[q] >> 8) & 0xff, cc = path[q] >> 16;
                        pv[q] = val[l][cc];
                        drop(l, bb, cc);
                    }
                    for (int q = 0; q < np; ++q) {
                        const int l = path[q] & 0xff, bb = (path[q] >> 8) & 0xff, cc = path[q] >> 16;
                        put(l, bb, cc == ca ? cb : ca, pv[q]);
                    }
                    c = ca;
                }
                put(u, b, c, (((v & 0x7fffffffu) - j0) * 4u) | (v & 0x80000000u));
            }
          }
        }
        // Concentrate the conflicts.  A step is a 2-way conflict iff it holds
        // an overflow vbank (b + 32k, k >= 1) edge, so the wavefronts are L +
        // |colours used by overflow vbanks|; the lower bound is L + K, K = the
        // largest overflow vbank (= the busiest bank's degree).  The Kempe
        // swaps above scatter those colours over all L steps (C3: 72% of the
        // steps conflicted, 1.72 wavefronts per LDS), so move every overflow
        // vbank's colours into [0, K): for its edge of colour x >= K pick a
        // y < K it lacks and swap x <-> y along the x/y path from it.  The
        // path enters vbanks by y and leaves by x, so it ends at any vbank
        // without x: a y whose path would end at an already aligned overflow
        // vbank is skipped (C3: 1.72 -> 1.60 wavefronts per LDS; the lower
        // bound, the busiest bank's degree / L, is ~1.35 -- reaching it needs
        // the conflict edges chosen first, a degree-bounded flow; not done).
        int K = 0;
        for (int vb = 32; vb < 32 * kGVB; ++vb) {
            int c = 0;
#pragma unroll
            for (int w = 0; w < kGCW; ++w) c += __popc(bmask[vb][w]);
            K = max(K, c);
        }
        uint32_t aligned[kGVB] = {};  // bit vb & 31 of word vb / 32
        auto has = [&](const uint32_t* msk, int c) { return (msk[c >> 5] >> (c & 31)) & 1u; };
        for (int vb = 32; K > 0 && K < C && vb < 32 * kGVB; ++vb) {
            for (int x = K; x < C; ++x) {
                if (!has(bmask[vb], x)) continue;
                for (int y = 0; y < K; ++y) {
                    if (has(bmask[vb], y)) continue;
                    int np = 0, xv = vb;
                    bool bad = false;
                    for (;;) {
                        const int l = bank_lane[xv][x];
                        if (l == 0xff) break;
                        path[np++] = (uint32_t)l | ((uint32_t)xv << 8) | ((uint32_t)x << 16);
                        const int v2 = lane_bank[l][y];
                        if (v2 == 0xff) break;
                        path[np++] = (uint32_t)l | ((uint32_t)v2 << 8) | ((uint32_t)y << 16);
                        if ((aligned[v2 >> 5] >> (v2 & 31)) & 1u) {
                            bad = true;  // would push an aligned vbank out of [0, K)
                            break;
                        }
                        xv = v2;
                    }
                    if (bad) continue;
                    for (int q = 0; q < np; ++q) {
                        const int l = path[q] & 0xff, bb = (path[q] >> 8) & 0xff, cc = path[q] >> 16;
                        pv[q] = val[l][cc];
                        drop(l, bb, cc);
                    }
                    for (int q = 0; q < np; ++q) {
                        const int l = path[q] & 0xff, bb = (path[q] >> 8) & 0xff, cc = path[q] >> 16;
                        put(l, bb, cc == x ? y : x, pv[q]);
                    }
                    break;
                }
            }
            aligned[vb >> 5] |= 1u << (vb & 31);
        }
    }
    __syncwarp();
    for (int t = 0; t < T; ++t) {
        const int b = t < C ? lane_bank[lane][t] : 0xff;
        const bool has = b != 0xff;
        const uint32_t used = __reduce_or_sync(0xffffffffu, has ? 1u << (b & 31) : 0u);
        const unsigned idle = __ballot_sync(0xffffffffu, !has);
        uint32_t w;
        if (has) {
            w = val[lane][t];
        } else {  // a zero word in the rank-th unused bank
            const int rank = __popc(idle & ((1u << lane) - 1u));
            w = (zero_word + (uint32_t)__fns(~used, 0, rank + 1)) * 4u;
        }
        sched[((int64_t)wg * kGTMax + t) * 32 + lane] = w;
    }
    if (lane == 0) tw[wg] = T;
}

// ---- the gather ----------------------------------------------------------------
// Acc = float: the fp32 sketch of the range finder.  Acc = double: the same
// gather with fp64 accumulation and an fp64 output (the fp32 entries and their
// +-1 signs are exact in fp64, the 1/sqrt(s) scale is applied once), for the
// psd Nystrom core, whose literal power W~^q Omega (cond ~1e15) turns the
// rounding of an fp32 sketch into a 1e-3 change of its error.
template <int NB, typename Acc = float, int TR = kGTReg>
__global__ void __maxnreg__(72)
sketch_gather_kernel(const float* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                     const int32_t* __restrict__ lanepos, int P, const uint32_t* __restrict__ sched,
                     const int32_t* __restrict__ tw, const int32_t* __restrict__ plan_fail,
                     Acc scale, Acc* __restrict__ out, int64_t ldo,
                     int64_t* nonfinite, uint32_t* __restrict__ amax, int accumulate,
                     int mark_fail) {
    extern __shared__ __align__(128) unsigned char sm[];
    if (*plan_fail) {
        // the plan's schedule overflowed: report it through the non-finite
        // counter (the caller re-runs with K2 v1; no host sync at plan time)
        if (blockIdx.x == 0 && threadIdx.x == 0 && nonfinite && mark_fail)
            atomicAdd(reinterpret_cast<unsigned long long*>(nonfinite), kGPlanFailMark);
        return;
    }
    constexpr uint32_t kB = GBuf<NB>::bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NB * (size_t)kB);
    uint32_t* done = reinterpret_cast<uint32_t*>(full + NB);  // warps finished with a buffer

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slice = blockIdx.x % P;
    const int g = blockIdx.x / P, G = gridDim.x / P;
    const uint32_t base = g_smem_u32(sm);
    const uint32_t zero_word = (uint32_t)((n + 31) / 32 * 32);
    const uint32_t row_bytes = (uint32_t)((n + 3) / 4 * 16);

    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; ++b) {
            g_mbar_init(&full[b], 1);
            done[b] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32 * NB) {  // zero words (targets of idle lanes) of every buffer
        float* z = reinterpret_cast<float*>(sm + (threadIdx.x >> 5) * (size_t)kB);
        z[zero_word + (threadIdx.x & 31)] = 0.f;
    }
    __syncthreads();
    if (warp == 0) {  // first NB rows of this group
        for (int b = 0; b < NB; ++b)
            if (g + b * (int64_t)G < m)
                g_bulk_load_e(base + b * kB, A + (g + b * (int64_t)G) * lda, row_bytes, &full[b]);
    }

    // compute warps: this warp's schedule -> registers (absolute smem addresses)
    const int wg = slice * kGW + warp;
    const int T = tw[wg];
    uint32_t e[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
        const uint32_t v =
            t < T ? __ldg(sched + ((int64_t)wg * kGTMax + t) * 32 + lane) : zero_word * 4u;
        // (steps >= TR, if any, are read per row below)
        e[t] = v + base;  // absolute smem address in buffer 0; bit 31 (sign) kept
    }
    const int lp = lanepos[(int64_t)wg * 32 + lane];
    const int64_t v_out = lp & (kGPrimary - 1);  // output position
    const bool valid = lp >= 0;                  // (second halves of split columns: no write)
    const bool primary = lp >= 0 && (lp & kGPrimary);
    bool bad = false;  // a non-finite output of this thread (iff a non-finite input)
    uint32_t mx = 0;   // max |output| (bits; non-negative floats order as integers)

    auto do_row = [&](int64_t i, int b, uint32_t ph, auto boff_c) {
        constexpr uint32_t boff = decltype(boff_c)::value;
        // (column passes after the first: the earlier sums towards the L1 now,
        // see the pair kernel)
        if (accumulate && valid) asm volatile("prefetch.global.L1 [%0];" ::"l"(out + i * ldo + v_out));
        g_mbar_wait(&full[b], ph);
        // opaque per row: stops the compiler from hoisting the per-entry masks
        // out of the row loop (3x the registers, spills) and orders the loads
        // below after the wait
#pragma unroll
        for (int t = 0; t < TR; ++t) asm volatile("" : "+r"(e[t]));
        Acc acc = 0;
#pragma unroll
        for (int t4 = 0; t4 < TR; t4 += 4) {
            if (t4 >= T) break;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t ev = e[t4 + u];
                float x;  // buffer offset as the LDS immediate
                asm("ld.shared.f32 %0, [%1+%2];" : "=f"(x) : "r"(ev & 0x7fffffffu), "n"(boff));
                acc += (Acc)__int_as_float(__float_as_int(x) ^ (int)(ev & 0x80000000u));
            }
        }
        // rare heavy warps: the steps past the register-resident ones stream
        // from the (L1-resident) schedule
        for (int t = TR; t < T; ++t) {
            const uint32_t ev = __ldg(sched + ((int64_t)wg * kGTMax + t) * 32 + lane) + base;
            float x;
            asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(x) : "r"(ev & 0x7fffffffu), "n"(boff));
            acc += (Acc)__int_as_float(__float_as_int(x) ^ (int)(ev & 0x80000000u));
        }
        // every load of this row (the non-volatile register-resident ones
        // included: acc depends on all of them) completes before this warp
        // reports the buffer done -- the last warp's refill overwrites it
        if constexpr (sizeof(Acc) == 4) asm volatile("" : "+f"(acc)::"memory");
        else asm volatile("" : "+d"(acc)::"memory");
        __syncwarp();
        if (lane == 0) {
            // the last warp done with this buffer refills it with row i + NB*G
            // (atom.inc wraps to 0 by itself; see the pair kernel)
            uint32_t finished;
            asm volatile("atom.shared.inc.u32 %0, [%1], %2;"
                         : "=r"(finished)
                         : "r"(g_smem_u32(&done[b])), "n"(kGW - 1)
                         : "memory");
            if (finished == kGW - 1) {
                const int64_t nx = i + NB * (int64_t)G;
                if (nx < m) {
                    asm volatile(
                        "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                            g_smem_u32(&full[b])),
                        "r"(row_bytes)
                        : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
                        "[%1], %2, [%3];" ::"r"(base + (uint32_t)b * kB),
                        "l"(reinterpret_cast<uint64_t>(A + nx * lda)), "r"(row_bytes),
                        "r"(g_smem_u32(&full[b]))
                        : "memory");
                }
            }
        }
        // a split column's second half sits on the next lane
        const Acc part = __shfl_down_sync(0xffffffffu, acc, 1);
        if (primary) acc += part;
        if (valid) {
            // column passes after the first add to what the earlier ones wrote
            const Acc o = accumulate ? fma(acc, scale, out[i * ldo + v_out]) : acc * scale;
            bad |= !isfinite(o);
            if constexpr (sizeof(Acc) == 4) mx = max(mx, __float_as_uint(fabsf(o)));
            out[i * ldo + v_out] = o;
        }
    };

    // one row body per buffer: the buffer offset is the LDS immediate
    uint32_t ph = 0;  // the k-th use of a buffer waits for parity k & 1
    for (int64_t i = g; i < m; i += NB * (int64_t)G, ph ^= 1u) {
        do_row(i, 0, ph, std::integral_constant<uint32_t, 0>());
        if (i + G < m) do_row(i + G, 1, ph, std::integral_constant<uint32_t, kB>());
        if constexpr (NB > 2)
            if (i + 2 * (int64_t)G < m)
                do_row(i + 2 * G, 2, ph, std::integral_constant<uint32_t, 2 * kB>());
    }

    if (amax) {  // max |A~| for the 3xFP16 split of A~ (skp_split_h2_f32, have_amax)
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0 && mx) atomicMax(amax, mx);
    }
    if (nonfinite) {
        const unsigned nb = __popc(__ballot_sync(0xffffffffu, bad));
        if (lane == 0 && nb)
            atomicAdd(reinterpret_cast<unsigned long long*>(nonfinite), (unsigned long long)nb);
    }
}

// {a0, a1} += {b0, b1} as one packed fp32x2 add (sm_100: FADD2), rounding as two FADDs
__device__ __forceinline__ void g_add2(float& a0, float& a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb;\n\t"
        "mov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %3};\n\t"
        "add.rn.f32x2 ra, ra, rb;\n\t"
        "mov.b64 {%0, %1}, ra;\n\t}"
        : "+f"(a0), "+f"(a1)
        : "f"(b0), "f"(b1));
}

// ---- K2 v3: two slices per CTA on a 16-bit schedule ----------------------------
// What binds K2 at C5 is the row ingest: every one of the P slice CTAs of a
// row group bulk-copies the whole row, and one SM receives ~150 GB/s however
// many CTAs read the row (profiles/r02w_k2_ingest.txt: 40 ms of a 78 ms pass
// at P = 10).  Here one CTA gathers two slices of the same plan from one copy
// of the row, halving the ingest; the schedule of both fits the registers of
// one because a pass of <= 16384 words needs 16-bit offsets: two entries per
// register.  Entry at an even step: low half, byte offset - 128 in bits 2..15,
// negate in bit 0; odd step: high half (bits 18..31), negate in bit 1.  Decode:
//     even: LOP3 (w & 0xfffc) -> LDS -> LEA (x + (w << 31)) -> FADD
//     odd:  SHR (w >> 16)     -> LDS -> SHL, LOP3 (sign)    -> FADD
// and the two slices step together, so the two FADDs of a step are one packed
// fp32x2 add (FADD2) on the accumulator pair: 4.0 instructions per entry
// (4.5 with scalar adds: C5 150.5 -> 142.3 ms, C3 10.65 -> 10.08 ms alone).
// The LDS immediate carries the buffer's absolute shared address SB + boff +
// 128, so SB -- the dynamic shared memory base, after the reserved words --
// is a template parameter, probed once by the launcher.  The window [128, 128 + 65532] holds the row
// from word 32 on and every zero word; an entry on one of the row's first 32
// words is replaced by the zero word of its bank (no new conflict) and
// gathered after the main steps (C3: ~1.5
// such entries per warp and slice) from a per-lane table in shared memory.
constexpr int kG3TR = 40;  // register-resident steps per slice (20 registers each)
constexpr int kG3Heads = 8;  // head entries per lane (shared-memory table)
// two row buffers; three of 65664 bytes (16384 + 32 words) fit beside the
// head table and were measured slower (C3 8.79 -> 9.24 ms, C5 121.0 -> 122.8
// ms alone): the row loop is issue-bound, not waiting on the refill
constexpr int kG3NB = 2;
constexpr uint32_t kG3B = kGBufBytes;
constexpr size_t kG3BufSmem = kG3NB * (size_t)kG3B + 64;
constexpr size_t kG3Smem = kG3BufSmem + (size_t)kG3Heads * kGThreads * 4;
template <uint32_t SB, bool ACC>
__global__ void __maxnreg__(72)
sketch_gather_pair_kernel(const float* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                          const int32_t* __restrict__ lanepos, int P2,
                          const uint32_t* __restrict__ sched, const int32_t* __restrict__ tw,
                          const int32_t* __restrict__ plan_fail, float scale,
                          float* __restrict__ out, int64_t ldo, int64_t* nonfinite,
                          uint32_t* __restrict__ amax, int mark_fail) {
    // ACC: a column pass after the first adds to what the earlier ones wrote
    extern __shared__ __align__(128) unsigned char sm[];
    if (*plan_fail) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && nonfinite && mark_fail)
            atomicAdd(reinterpret_cast<unsigned long long*>(nonfinite), kGPlanFailMark);
        return;
    }
    constexpr int TRK = kG3TR, RK = TRK / 2;
    constexpr uint32_t kB = kG3B;
    constexpr int NB = kG3NB;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NB * (size_t)kB);
    uint32_t* done = reinterpret_cast<uint32_t*>(full + NB);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sg = blockIdx.x % P2;
    const int g = blockIdx.x / P2, G = gridDim.x / P2;
    const uint32_t base = g_smem_u32(sm);  // == SB
    const uint32_t zero_word = (uint32_t)((n + 31) / 32 * 32);
    const uint32_t row_bytes = (uint32_t)((n + 3) / 4 * 16);

    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; ++b) {
            g_mbar_init(&full[b], 1);
            done[b] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32 * NB) {
        float* z = reinterpret_cast<float*>(sm + (threadIdx.x >> 5) * (size_t)kB);
        z[zero_word + (threadIdx.x & 31)] = 0.f;
    }
    __syncthreads();
    if (warp == 0) {
        for (int b = 0; b < NB; ++b)
            if (g + b * (int64_t)G < m)
                g_bulk_load_e(base + b * kB, A + (g + b * (int64_t)G) * lda, row_bytes, &full[b]);
    }

    // both slices' schedules -> packed registers; head entries -> this
    // thread's column of the head table after the barriers (absolute
    // address, bit 31 negate, bit 30 = slice 1; idle slots: a zero word)
    const int wg0 = (2 * sg) * kGW + warp, wg1 = wg0 + kGW;
    const int T0 = tw[wg0], T1 = tw[wg1];
    const int TM = max(T0, T1);
    uint32_t e[2 * RK];
    uint32_t* heads = reinterpret_cast<uint32_t*>(sm + kG3BufSmem);
#pragma unroll
    for (int q = 0; q < kG3Heads; ++q) heads[q * kGThreads + threadIdx.x] = (zero_word + lane) * 4u + base;
    int nhd = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int wgk = k ? wg1 : wg0, Tk = k ? T1 : T0;
#pragma unroll
        for (int t = 0; t < TRK; ++t) {
            uint32_t v = t < Tk ? __ldg(sched + ((int64_t)wgk * kGTMax + t) * 32 + lane)
                                : zero_word * 4u;
            uint32_t off = v & 0x7fffffffu, neg = v >> 31;
            if (t < Tk && off < 128u) {  // one of the row's first 32 words
                const uint32_t h = (off + base) | (neg << 31) | ((uint32_t)k << 30);
                if (nhd < kG3Heads) heads[nhd * kGThreads + threadIdx.x] = h;
                ++nhd;
                off = zero_word * 4u + off;  // the zero word of the same bank
                neg = 0;
            }
            const uint32_t h16 = off - 128u;
            if ((t & 1) == 0) e[k * RK + t / 2] = h16 | neg;
            else e[k * RK + t / 2] |= (h16 << 16) | (neg << 1);
        }
    }
    // heads: up to kG3Heads per lane from the table (C3/C5: at most 3; two
    // columns of one lane share the ~256 head entries of a pass); a warp with
    // more re-reads its schedule for them every row
    const int HT = __reduce_max_sync(0xffffffffu, (unsigned)nhd);
    const bool head_scan = HT > kG3Heads;
    int lp = lanepos[(int64_t)wg0 * 32 + lane];
    const int32_t v_out0 = lp & (kGPrimary - 1);
    const bool valid0 = lp >= 0, primary0 = lp >= 0 && (lp & kGPrimary);
    lp = lanepos[(int64_t)wg1 * 32 + lane];
    const int32_t v_out1 = lp & (kGPrimary - 1);
    const bool valid1 = lp >= 0, primary1 = lp >= 0 && (lp & kGPrimary);
    uint32_t mx = 0;

    auto do_row = [&](int64_t i, int b, uint32_t ph, auto boff_c) {
        constexpr uint32_t boff = decltype(boff_c)::value;
        constexpr uint32_t imm = SB + boff + 128u;
        // the barrier, the done count and the buffer of this row body at their
        // absolute shared addresses (SB is a template parameter): no address
        // arithmetic from the shared window base in the row loop
        constexpr uint32_t kFull = SB + NB * kB + 8u * (boff / kB);
        constexpr uint32_t kDone = SB + NB * kB + 8u * NB + 4u * (boff / kB);
        // a column pass after the first adds to the sums the earlier passes
        // wrote: ask for them now, or every warp of the CTA meets their DRAM
        // latency together at the end of the row (C5: pass 2 ran 89 ms against
        // 63 ms for pass 1; K2 alone 131.3 -> 121.3 ms with the prefetch)
        if constexpr (ACC) {
            float* pr = out + i * ldo;  // (the next row's instead: the same, 121 ms)
            if (valid0) asm volatile("prefetch.global.L1 [%0];" ::"l"(pr + v_out0));
            if (valid1) asm volatile("prefetch.global.L1 [%0];" ::"l"(pr + v_out1));
        }
        g_mbar_wait_a(kFull, ph);
#pragma unroll
        for (int t = 0; t < 2 * RK; ++t) asm volatile("" : "+r"(e[t]));
        float acc[2] = {0.f, 0.f};
        // both slices step together: their two accumulators are one packed
        // fp32x2 add per step pair (the steps past a slice's own length read
        // its zero word); per slice the order of the sum is unchanged
#pragma unroll
        for (int t4 = 0; t4 < TRK; t4 += 4) {
            if (t4 >= TM) break;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t w0 = e[t4 / 2 + u], w1 = e[RK + t4 / 2 + u];
                float x0, y0, x1, y1;
                asm("ld.shared.f32 %0, [%1+%2];" : "=f"(x0) : "r"(w0 & 0xfffcu), "n"(imm));
                asm("ld.shared.f32 %0, [%1+%2];" : "=f"(x1) : "r"(w1 & 0xfffcu), "n"(imm));
                asm("ld.shared.f32 %0, [%1+%2];" : "=f"(y0) : "r"(w0 >> 16), "n"(imm));
                asm("ld.shared.f32 %0, [%1+%2];" : "=f"(y1) : "r"(w1 >> 16), "n"(imm));
                g_add2(acc[0], acc[1], __int_as_float(__float_as_int(x0) + (int)(w0 << 31)),
                       __int_as_float(__float_as_int(x1) + (int)(w1 << 31)));
                g_add2(acc[0], acc[1],
                       __int_as_float(__float_as_int(y0) ^ (int)((w0 << 30) & 0x80000000u)),
                       __int_as_float(__float_as_int(y1) ^ (int)((w1 << 30) & 0x80000000u)));
            }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int Tk = k ? T1 : T0;
            const int wgk = k ? wg1 : wg0;
            for (int t = TRK; t < Tk; ++t) {  // heavy warps: the rest from L1
                const uint32_t ev = __ldg(sched + ((int64_t)wgk * kGTMax + t) * 32 + lane) + base;
                float x;
                asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(x) : "r"(ev & 0x7fffffffu), "n"(boff));
                acc[k] += __int_as_float(__float_as_int(x) ^ (int)(ev & 0x80000000u));
            }
        }
        if (!head_scan) {
            for (int q = 0; q < HT; ++q) {
                const uint32_t h = heads[q * kGThreads + threadIdx.x];
                float x;
                asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(x) : "r"(h & 0x3fffffffu), "n"(boff));
                x = __int_as_float(__float_as_int(x) ^ (int)(h & 0x80000000u));
                if (h & 0x40000000u) acc[1] += x;
                else acc[0] += x;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int wgk = k ? wg1 : wg0, Tk = k ? T1 : T0;
                for (int t = 0; t < min(Tk, TRK); ++t) {
                    const uint32_t v = __ldg(sched + ((int64_t)wgk * kGTMax + t) * 32 + lane);
                    if ((v & 0x7fffffffu) >= 128u) continue;
                    float x;
                    asm volatile("ld.shared.f32 %0, [%1+%2];"
                                 : "=f"(x) : "r"((v & 0x7fffffffu) + base), "n"(boff));
                    acc[k] += __int_as_float(__float_as_int(x) ^ (int)(v & 0x80000000u));
                }
            }
        }
        asm volatile("" : "+f"(acc[0]), "+f"(acc[1])::"memory");
        __syncwarp();
        if (lane == 0) {
            // atom.inc wraps to 0 at the last warp by itself; an atom.add here
            // (atomicAdd, or inline) is turned into a warp-aggregated add by
            // ptxas, ~18 instructions per row and warp
            uint32_t finished;
            asm volatile("atom.shared.inc.u32 %0, [%1], %2;"
                         : "=r"(finished)
                         : "r"(kDone), "n"(kGW - 1)
                         : "memory");
            if (finished == kGW - 1) {
                const int64_t nx = i + NB * (int64_t)G;
                if (nx < m) {
                    asm volatile(
                        "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(kFull),
                        "r"(row_bytes)
                        : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
                        "[%1], %2, [%3];" ::"r"(SB + boff),
                        "l"(reinterpret_cast<uint64_t>(A + nx * lda)), "r"(row_bytes), "r"(kFull)
                        : "memory");
                }
            }
        }
        float* prow = out + i * ldo;  // one 64-bit product per row, not per slice
        asm volatile("" : "+l"(prow));  // (opaque: or it is recomputed per slice)
        __builtin_assume(__isGlobal(prow));
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const float part = __shfl_down_sync(0xffffffffu, acc[k], 1);
            if (k ? primary1 : primary0) acc[k] += part;
            if (k ? valid1 : valid0) {
                float* po = prow + (k ? v_out1 : v_out0);
                const float o = ACC ? fmaf(acc[k], scale, *po) : acc[k] * scale;
                mx = max(mx, __float_as_uint(fabsf(o)));  // (inf, nan: the largest patterns)
                *po = o;
            }
        }
    };

    uint32_t ph = 0;
    for (int64_t i = g; i < m; i += NB * (int64_t)G, ph ^= 1u) {
        do_row(i, 0, ph, std::integral_constant<uint32_t, 0>());
        if (i + G < m) do_row(i + G, 1, ph, std::integral_constant<uint32_t, kB>());
        if constexpr (NB > 2)
            if (i + 2 * (int64_t)G < m)
                do_row(i + 2 * G, 2, ph, std::integral_constant<uint32_t, 2 * kB>());
    }

    // a non-finite output of this thread (iff a non-finite input): its |.|
    // pattern is the largest there is, so the running max holds it
    const bool bad = mx >= 0x7f800000u;
    if (amax) {
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0 && mx) atomicMax(amax, mx);
    }
    if (nonfinite) {
        const unsigned nb = __popc(__ballot_sync(0xffffffffu, bad));
        if (lane == 0 && nb)
            atomicAdd(reinterpret_cast<unsigned long long*>(nonfinite), (unsigned long long)nb);
    }
}

// the dynamic shared memory base of a kernel without static shared memory
__global__ void smem_base_probe_kernel(uint32_t* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    if (threadIdx.x == 0) *out = g_smem_u32(sm);
}

// apply_right in the reference's column order: X[i, perm[v]] = X[i, v] in
// place (X = the permuted A S P written by the gather).  One CTA holds the
// inverse permutation and one row in shared memory: coalesced row read,
// coalesced permuted write.  HBM-bound (2 x rows x cols words).
template <typename T>
__global__ void __launch_bounds__(512)
unpermute_cols_kernel(T* __restrict__ X, int64_t rows, int cols, int64_t ldx,
                      const int32_t* __restrict__ perm) {
    extern __shared__ __align__(16) unsigned char usm[];
    int32_t* inv = reinterpret_cast<int32_t*>(usm);
    T* row = reinterpret_cast<T*>(usm + ((size_t)cols * 4 + 15) / 16 * 16);
    for (int v = threadIdx.x; v < cols; v += blockDim.x) inv[perm[v]] = v;
    for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
        __syncthreads();  // inv built / the previous row written out
        T* x = X + i * ldx;
        for (int v = threadIdx.x; v < cols; v += blockDim.x) row[v] = x[v];
        __syncthreads();
        for (int c = threadIdx.x; c < cols; c += blockDim.x) x[c] = row[inv[c]];
    }
}

}  // namespace

// plan layout (bytes): perm int32[P*kGCols] | fail int32 | pad to 16 |
//   per column pass h < H: tw int32[P*kGW] (padded to 16) | sched uint32[P*kGW*kGTMax*32]
//   | seg_beg int32[H][P*kGCols] | seg_cnt int32[H][P*kGCols] | lanepos int32[P*kGCols]
// H = ceil(n / 24576) column passes of npass (a multiple of 32) columns each.
// slices of at most kGCols - 96 columns: the spare lanes split heavy columns
// (with none, C3-like sketches put 56 steps on the heaviest warps, past the 44
// register-resident ones); C3's 4000 columns -> 5 x 800
constexpr int kGSpare = 96;
// (an even count above one slice: K2 v3 pairs the slices)
int gather_slices(int64_t r) {
    const int p = (int)cdiv(r, (int64_t)(kGCols - kGSpare));
    return p > 1 ? (p + 1) / 2 * 2 : p;
}
// balanced slice width: the P slices share the r columns evenly (multiple of
// 32), so no CTA carries a short last slice while its SM idles (C3: 6 x 672
// instead of 5 x 768 + 160)
int gather_width(int64_t r) {
    return (int)(cdiv(cdiv(r, (int64_t)gather_slices(r)), 32) * 32);
}
int gather_passes(int64_t n) { return (int)cdiv(n, (int64_t)(kGBufWords - 32)); }
int gather_npass(int64_t n) {
    return (int)(cdiv(cdiv(n, (int64_t)gather_passes(n)), 32) * 32);
}

struct GLayout {
    int P, H, npass;
    int32_t* perm;
    int32_t* fail;
    GSched ps;
    int32_t* seg_beg;
    int32_t* seg_cnt;
    int32_t* lanepos;
    int64_t bytes;
};
GLayout gather_layout(void* plan, int64_t n, int64_t r) {
    GLayout L;
    L.P = gather_slices(r);
    L.H = gather_passes(n);
    L.npass = gather_npass(n);
    char* b = reinterpret_cast<char*>(plan);
    int64_t off = 0;
    auto take = [&](int64_t bytes) {
        char* p = b ? b + off : nullptr;
        off += (bytes + 15) / 16 * 16;
        return p;
    };
    L.perm = reinterpret_cast<int32_t*>(take((int64_t)L.P * kGCols * 4));
    L.fail = reinterpret_cast<int32_t*>(take(4));
    L.ps.H = L.H;
    for (int h = 0; h < kGMaxPass; ++h) {
        L.ps.tw[h] = nullptr;
        L.ps.sched[h] = nullptr;
    }
    for (int h = 0; h < L.H && h < kGMaxPass; ++h) {
        L.ps.tw[h] = reinterpret_cast<int32_t*>(take((int64_t)L.P * kGW * 4));
        L.ps.sched[h] = reinterpret_cast<uint32_t*>(take((int64_t)L.P * kGW * kGTMax * 32 * 4));
    }
    L.seg_beg = reinterpret_cast<int32_t*>(take((int64_t)L.H * L.P * kGCols * 4));
    L.seg_cnt = reinterpret_cast<int32_t*>(take((int64_t)L.H * L.P * kGCols * 4));
    L.lanepos = reinterpret_cast<int32_t*>(take((int64_t)L.P * kGCols * 4));
    L.bytes = off;
    return L;
}
int64_t gather_plan_bytes(int64_t n, int64_t r) { return gather_layout(nullptr, n, r).bytes; }

int gather_plan(const int32_t* colptr, const int32_t* entries, int64_t n, int64_t r, void* plan,
                int64_t plan_bytes, cudaStream_t st) {
    SKP_ARG(n >= 1 && r >= 1 && plan, "sketch_gather_plan: bad sizes");
    if (gather_passes(n) > kGMaxPass) {
        set_error("unsupported: sketch_gather needs n <= %d", kGMaxPass * (kGBufWords - 32));
        return SKP_ERR_UNSUPPORTED;
    }
    SKP_ARG(plan_bytes >= gather_plan_bytes(n, r), "sketch_gather_plan: plan buffer too small");
    const GLayout L = gather_layout(plan, n, r);
    SKP_CUDA(cudaMemsetAsync(L.fail, 0, 4, st));
    const int width = gather_width(r);
    gather_sort_kernel<<<L.P, 256, 0, st>>>(colptr, entries, r, width, (int64_t)L.P * kGCols, L.H,
                                            L.npass, L.perm, L.seg_beg, L.seg_cnt, L.lanepos,
                                            L.fail);
    SKP_LAUNCHED(gather_sort_kernel);
    const int nw = L.P * kGW;
    gather_sched_kernel<<<(unsigned)(nw * L.H), 32, 0, st>>>(
        L.seg_beg, L.seg_cnt, entries, nw, n, L.npass, L.ps, L.fail);
    SKP_LAUNCHED(gather_sched_kernel);
    return SKP_OK;
}

// dynamic shared memory base address on device `dev` (probed once; -1 on error)
int smem_base(int dev, size_t smem) {
    static int cached[64];
    static bool have[64];
    if (dev < 0 || dev >= 64) return -1;
    if (have[dev]) return cached[dev];
    uint32_t* d = nullptr;
    uint32_t h = 0xffffffffu;
    int rc = -1;
    if (cudaFuncSetAttribute(smem_base_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) == cudaSuccess &&
        cudaMalloc(&d, 4) == cudaSuccess) {
        smem_base_probe_kernel<<<1, 32, smem>>>(d);
        if (cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost) == cudaSuccess) rc = (int)h;
        cudaFree(d);
    }
    cudaGetLastError();
    cached[dev] = rc;
    have[dev] = true;
    return rc;
}

template <typename Acc>
int sketch_gather(const float* A, int64_t lda, int64_t m, int64_t n, int64_t r,
                      const void* plan, Acc scale, Acc* out, int64_t ldo, double* fro2,
                      int64_t* nonfinite, uint32_t* amax, cudaStream_t st) {
    SKP_ARG(m >= 0 && n >= 1 && r >= 1 && ldo >= r, "sketch_gather: bad sizes");
    if (gather_passes(n) > kGMaxPass || (reinterpret_cast<uintptr_t>(A) & 15) || (lda & 3) ||
        lda < (n + 3) / 4 * 4) {
        set_error("unsupported: sketch_gather needs n <= %d and 16-byte aligned, padded rows",
                  kGMaxPass * (kGBufWords - 32));
        return SKP_ERR_UNSUPPORTED;
    }
    if (m == 0) return SKP_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const GLayout L = gather_layout(const_cast<void*>(plan), n, r);
    const int P = L.P;
    const int G = std::max(1, std::min<int>(sms / P, (int)std::min<int64_t>(m, 1 << 20)));
    // fp64 accumulation: 40 register-resident steps (the accumulator and the
    // output take two registers more)
    auto kern = sizeof(Acc) == 4 ? sketch_gather_kernel<2, Acc, kGTReg> : sketch_gather_kernel<2, Acc, 40>;
    const size_t smem = GBuf<2>::smem;
    // K2 v3 (two slices per CTA) for fp32 passes of <= 16384 words
    if constexpr (sizeof(Acc) == 4) {
        const int sb = P % 2 == 0 && L.npass <= 16384 ? smem_base(dev, smem) : -1;
        auto pk0 = sb == 0      ? sketch_gather_pair_kernel<0, false>
                   : sb == 1024 ? sketch_gather_pair_kernel<1024, false>
                                : nullptr;
        auto pk1 = sb == 0 ? sketch_gather_pair_kernel<0, true> : sketch_gather_pair_kernel<1024, true>;
        if (pk0) {
            const int P2 = P / 2;
            const int G2 = std::max(1, std::min<int>(sms / P2, (int)std::min<int64_t>(m, 1 << 20)));
            SKP_CUDA(cudaFuncSetAttribute(pk0, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kG3Smem));
            SKP_CUDA(cudaFuncSetAttribute(pk1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kG3Smem));
            // Row chunks: the P2 CTAs of a row group copy the same rows, and only
            // the first copy of a row should come from DRAM; left to themselves
            // they drift apart by more rows than the L2 holds (C5: 253 GB read
            // per pass for 69 GB of A).  Any coupling inside the kernel cost
            // more than it saved (profiles/r02zc_k2_pacing_ab.txt); a kernel
            // boundary every 512 row steps re-aligns them for ~15 us: C5 118.0
            // -> 113.3 ms (flat from 384 to 1024 row steps; 128: 122.4 ms).  With
            // P2 = 3 (C3) there is nothing to gain (8.75 -> 8.90 ms): one launch.
            const int64_t chunk_rows = (int64_t)G2 * 512;
            const int64_t chunk = (P2 >= 4 && m >= 8 * chunk_rows) ? chunk_rows : m;
            for (int h = 0; h < L.H; ++h) {
                const int64_t j0 = (int64_t)h * L.npass, nh = std::min<int64_t>(L.npass, n - j0);
                const bool last = h + 1 == L.H;
                for (int64_t r0 = 0; r0 < m; r0 += chunk) {
                    (h > 0 ? pk1 : pk0)<<<G2 * P2, kGThreads, kG3Smem, st>>>(
                        A + j0 + r0 * lda, lda, std::min(chunk, m - r0), nh, L.lanepos, P2,
                        L.ps.sched[h], L.ps.tw[h], L.fail, scale, out + r0 * ldo, ldo,
                        last ? nonfinite : (h == 0 ? nonfinite : nullptr), last ? amax : nullptr,
                        h == 0 && r0 == 0);
                    SKP_LAUNCHED(sketch_gather_pair_kernel);
                }
            }
            if (fro2) return skp_sumsq_f32(A, m, n, lda, fro2, nullptr, st);
            return SKP_OK;
        }
    }
    SKP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // one launch per column pass: pass h gathers A[:, h*npass ...] and adds
    // to what the earlier passes wrote; the checks ride on the last pass
    for (int h = 0; h < L.H; ++h) {
        const int64_t j0 = (int64_t)h * L.npass, nh = std::min<int64_t>(L.npass, n - j0);
        const bool last = h + 1 == L.H;
        kern<<<G * P, kGThreads, smem, st>>>(
            A + j0, lda, m, nh, L.lanepos, P, L.ps.sched[h], L.ps.tw[h], L.fail, scale, out, ldo,
            last ? nonfinite : (h == 0 ? nonfinite : nullptr), last ? amax : nullptr, h > 0,
            h == 0);
        SKP_LAUNCHED(sketch_gather_kernel);
    }
    if (fro2) {  // ||A||_F^2: a separate HBM-bound pass (only when asked for)
        const int rc = skp_sumsq_f32(A, m, n, lda, fro2, nullptr, st);
        if (rc != SKP_OK) return rc;
    }
    return SKP_OK;
}

template <typename T>
int unpermute_cols(T* X, int64_t rows, int64_t cols, int64_t ldx, const int32_t* perm,
                   cudaStream_t st) {
    SKP_ARG(rows >= 0 && cols >= 0 && ldx >= cols && (cols == 0 || perm), "unpermute_cols: bad sizes");
    const size_t smem = ((size_t)cols * 4 + 15) / 16 * 16 + (size_t)cols * sizeof(T);
    if (smem > 200 * 1024) {
        set_error("unsupported: unpermute_cols needs cols <= %d", (int)(200 * 1024 / (4 + sizeof(T))));
        return SKP_ERR_UNSUPPORTED;
    }
    if (!rows || !cols) return SKP_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    SKP_CUDA(cudaFuncSetAttribute(unpermute_cols_kernel<T>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int per_sm = std::max(1, std::min(4, (int)(220 * 1024 / smem)));
    const int64_t grid = std::min<int64_t>(rows, (int64_t)sms * per_sm);
    unpermute_cols_kernel<T><<<(unsigned)grid, 512, smem, st>>>(X, rows, (int)cols, ldx, perm);
    SKP_LAUNCHED(unpermute_cols_kernel);
    return SKP_OK;
}

}  // namespace skp

using namespace skp;

extern "C" int64_t skp_sketch_gather_plan_bytes(int64_t n, int64_t r) {
    return gather_plan_bytes(n, r);
}
extern "C" int64_t skp_sketch_gather_plan_fail_offset(int64_t r) {
    return (int64_t)gather_slices(r) * kGCols * 4;
}
extern "C" int skp_sketch_gather_plan(const int32_t* colptr, const int32_t* entries, int64_t n,
                                      int64_t r, void* plan, int64_t plan_bytes, void* stream) {
    return gather_plan(colptr, entries, n, r, plan, plan_bytes, (cudaStream_t)stream);
}
extern "C" int skp_sketch_gather_f32(const float* A, int64_t lda, int64_t m, int64_t n, int64_t r,
                                     const void* plan, float scale, float* out, int64_t ldo,
                                     double* fro2, int64_t* nonfinite, uint32_t* amax,
                                     void* stream) {
    return sketch_gather<float>(A, lda, m, n, r, plan, scale, out, ldo, fro2, nonfinite, amax,
                                (cudaStream_t)stream);
}
extern "C" int skp_sketch_gather_f32_acc64(const float* A, int64_t lda, int64_t m, int64_t n,
                                           int64_t r, const void* plan, double scale, double* out,
                                           int64_t ldo, double* fro2, int64_t* nonfinite,
                                           void* stream) {
    return sketch_gather<double>(A, lda, m, n, r, plan, scale, out, ldo, fro2, nonfinite, nullptr,
                                 (cudaStream_t)stream);
}
extern "C" int skp_unpermute_cols_f32(float* X, int64_t rows, int64_t cols, int64_t ldx,
                                      const int32_t* perm, void* stream) {
    return unpermute_cols<float>(X, rows, cols, ldx, perm, (cudaStream_t)stream);
}
extern "C" int skp_unpermute_cols_f64(double* X, int64_t rows, int64_t cols, int64_t ldx,
                                      const int32_t* perm, void* stream) {
    return unpermute_cols<double>(X, rows, cols, ldx, perm, (cudaStream_t)stream);
}
extern "C" int skp_sketch_gather_variant(int64_t n, int64_t r) {
    if (n < 1 || r < 1 || gather_passes(n) > kGMaxPass) return 0;
    int dev = 0;
    cudaGetDevice(&dev);
    const int sb = smem_base(dev, GBuf<2>::smem);
    return gather_slices(r) % 2 == 0 && gather_npass(n) <= 16384 && (sb == 0 || sb == 1024) ? 3 : 2;
}
