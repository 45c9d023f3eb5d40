// K4: FP32 GEMM on the sm_100a tensor cores by the 3xTF32 split, tcgen05/TMEM.
//
//   C = alpha * op(A) op(B) + beta * C,   a = a_hi + a_lo,
//   a.b ~= a_hi.b_hi + a_hi.b_lo + a_lo.b_hi   (error ~2^-20 relative per term,
//   below the fp32 accumulation error of the TMEM accumulator for K >~ 100)
// kind::tf32 reads fp32 containers and TRUNCATES to the TF32 grid (measured on
// B200: raw-operand products match truncated inputs to accumulation noise and
// miss round-to-nearest by ~500x), so a raw fp32 value IS its hi part and only
// lo = x - trunc(x) (exact in fp32) is materialised.
//
// The A operand lives in TENSOR MEMORY (tcgen05.mma A-from-TMEM): with both
// operands in shared memory the six MMAs of a stage re-read A and B from smem
// (60 KB/stage) and, with the TMA writes and the split, shared memory
// (128 B/clk) -- not the tensor pipe -- bounded the kernel.  Now the split
// warps read each A row once and store hi|lo straight into TMEM, and the MMAs
// only stream B from smem.
//
// One persistent CTA per SM, warp-specialised (14 warps):
//   warp 0      TMA producer: raw fp32 A and B tiles -> smem ring (BK = 32)
//   warp 1      MMA issuer: tcgen05.mma.kind::tf32 [acc], [A tmem], B desc,
//               12 per stage (4 K-steps x 3 products); owns the TMEM allocation
//   warps 2-5   A split: thread = tile row; smem row -> (hi, lo) -> tcgen05.st
//               into the stage's TMEM A slot (64 columns: 32 hi | 32 lo)
//   warps 6-9   B split: b_lo = b - trunc(b) beside each raw B tile in smem
//   warps 10-13 epilogue: tcgen05.ld 32x32b -> alpha/beta -> global (or split-K
//               partials), overlapping the next tile's main loop
// TMEM columns: [acc buffer 0 | acc buffer 1 | A slot 0..S-1].
// All issuing is warp-convergent (elect.sync inside the asm): a divergent
// `if (lane == 0)` issue path costs ~300 cycles per tcgen05/TMA instruction.
// Operands may be K-major or MN-major: B's UMMA descriptor carries its
// major-ness; A is re-laid row-per-lane by the split warps either way.
// Tiles: BM = 128 (UMMA M), BN = runtime multiple of 16 (32 for one-box MN
// loads) <= 192, BK = 32 (a stage carries 12 MMAs, ~1150 tensor cycles, so
// the per-stage barrier / TMA-issue / split costs stay off the critical path).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <stdlib.h>
#include <stdio.h>

#include "common.cuh"
#include "gemm.h"
#include "tc_ptx.cuh"

namespace skp {
namespace {

constexpr int BM = 128;
constexpr int BK = 32;
constexpr int kKSteps = BK / 8;      // tf32 UMMA K = 8
constexpr uint32_t kASlotCols = 2 * BK;  // TMEM columns per A slot: hi | lo
constexpr int kWarpTma = 0, kWarpMma = 1, kWarpAx = 2, kWarpBx = 6, kWarpEpi = 10, kNumEpi = 4;
constexpr int kNumXf = 8;  // A-split + B-split warps arriving on split[s]
constexpr int kMaxBn = 192;
constexpr int kThreads = 32 * (kWarpEpi + kNumEpi);
constexpr uint32_t kTmemCols = 512;
constexpr int kMaxStages = 12;

struct TcParams {
    int M, N, K;
    int bn, tiles_m, tiles_n, splits, kb_per_split, num_kb;
    int a_kmajor, b_kmajor;
    float alpha, beta;
    float* C;
    long long ldc;
    float* ws;
    int stages;
    uint32_t a_bytes, b_bytes, stage_bytes;
    uint32_t idesc;
    int a_mn3d, b_mn3d;  // MN-major operand loaded by ONE 3-D box per stage
    int acc_stride;      // TMEM columns per accumulator buffer
    int nacc;            // accumulator buffers (2: epilogue overlaps the next tile)
};

constexpr uint32_t kMnChunkBytes = 32 * BK * 4;  // one TMA box: 32 MN x BK K

__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int kmajor, int j) {
    return kmajor ? make_desc(base + 32u * j, 16u, 1024u, kLayoutSW128)
                  : make_desc(base + 1024u * j, kMnChunkBytes, 512u, kLayoutSW128Base32B);
}

struct Work {
    int tm, tn, ks, kb0, kb1;
};
__device__ __forceinline__ Work unit_of(const TcParams& p, int u) {
    // N-tiles of one M block are adjacent units -> co-resident CTAs share the
    // A row block through L2 (one DRAM read of A per M block)
    Work w;
    w.tn = u % p.tiles_n;
    int r = u / p.tiles_n;
    w.tm = r % p.tiles_m;
    w.ks = r / p.tiles_m;
    w.kb0 = w.ks * p.kb_per_split;
    w.kb1 = min(w.kb0 + p.kb_per_split, p.num_kb);
    return w;
}


// kPair: a CTA pair (cluster of 2, tcgen05 cta_group::2) computes a 256-row
// tile: each CTA holds its own 128 A rows (in its TMEM) and HALF of the B tile
// (bn/2 columns) in its smem; the leader's MMA warp issues M=256 MMAs that
// read both halves, so each SM streams ~30% fewer operand bytes from L2 and
// reads half as much B from smem.  Split / epilogue warps of both CTAs arrive
// on the leader's barriers; MMA commits multicast to both CTAs.
template <bool kPair>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const TcParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * p.stage_bytes);
    uint64_t* full = bars;
    uint64_t* split = bars + S;
    uint64_t* empty = bars + 2 * S;
    uint64_t* tfull = bars + 3 * S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int units = p.tiles_m * p.tiles_n * p.splits;
    const uint32_t rank = kPair ? cluster_rank() : 0u;
    const bool leader = rank == 0;
    const int ustart = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int ustride = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    constexpr int kRowsPerUnit = kPair ? 2 * BM : BM;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            // paired: the peer's split warps arrive locally and its MMA warp
            // forwards ONE cluster-scope arrive per stage to the leader (a
            // release.cluster arrive from every split warp cost ~1000 cycles/stage)
            mbar_init(&split[s], (kPair && leader) ? kNumXf + 1 : kNumXf);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kPair ? 2 * kNumEpi : kNumEpi);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kWarpMma) {
        if (kPair) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    if (kPair) cluster_sync_all();
    else __syncthreads();
    tc_fence_after();
    // arrival targets on the leader (own barriers when not paired)
    const uint32_t split_cl0 = kPair ? mapa_shared(smem_u32(split), 0) : 0u;
    const uint32_t tempty_cl0 = kPair ? mapa_shared(smem_u32(tempty), 0) : 0u;
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t acol0 = (uint32_t)(p.nacc * p.acc_stride);  // first A slot column

    // stage layout: [A raw (a_bytes) | B raw (b_bytes) | B lo (b_bytes)]
    const uint32_t smem0 = smem_u32(smem);
    auto stage_a = [&](int s) { return smem + (size_t)s * p.stage_bytes; };
    auto stage_b = [&](int s) { return stage_a(s) + p.a_bytes; };

    if (warp == kWarpTma) {
        Ring r;
        for (int u = ustart; u < units; u += ustride) {
            Work w = unit_of(p, u);
            const int m0 = w.tm * kRowsPerUnit + (int)rank * BM;
            const int n0 = w.tn * p.bn + (kPair ? (int)rank * (p.bn / 2) : 0);
            for (int kb = w.kb0; kb < w.kb1; ++kb, r.next(S)) {
                const int s = r.s;
                mbar_wait_k<kPair>(&empty[s], r.ph ^ 1);
                mbar_expect_tx_e(&full[s], p.a_bytes + p.b_bytes);
                const int k0 = kb * BK;
                const int k0b = k0;
                if (p.a_kmajor) {
                    tma_load_2d_e(&map_a, &full[s], stage_a(s), k0, m0);
                } else if (p.a_mn3d) {
                    tma_load_3d_e(&map_a, &full[s], stage_a(s), 0, k0, m0 / 32);
                } else {
                    for (int c = 0; c < BM / 32; ++c)
                        tma_load_2d_e(&map_a, &full[s], stage_a(s) + c * kMnChunkBytes, m0 + 32 * c,
                                      k0);
                }
                if (p.b_kmajor) {
                    tma_load_2d_e(&map_b, &full[s], stage_b(s), k0b, n0);
                } else if (p.b_mn3d) {
                    tma_load_3d_e(&map_b, &full[s], stage_b(s), 0, k0b, n0 / 32);
                } else {
                    const int bcols = kPair ? p.bn / 2 : p.bn;
                    for (int c = 0; c < (bcols + 31) / 32; ++c)
                        tma_load_2d_e(&map_b, &full[s], stage_b(s) + c * kMnChunkBytes, n0 + 32 * c,
                                      k0b);
                }
            }
        }
    } else if (warp == kWarpMma && leader) {
        // B descriptors: stage 0 / K-step 0, plus per-stage, per-K-step and
        // hi->lo offsets (the 14-bit start-address field never carries:
        // smem addresses < 228 KB)
        const uint64_t bdesc0 = operand_desc(smem_u32(stage_b(0)), p.b_kmajor, 0);
        const uint64_t sstep = p.stage_bytes >> 4;
        const uint64_t jstep = p.b_kmajor ? (32u >> 4) : (1024u >> 4);
        const uint64_t lostep = p.b_bytes >> 4;
        Ring r;
        int ul = 0;
        for (int u = ustart; u < units; u += ustride, ++ul) {
            Work w = unit_of(p, u);
            const int buf = p.nacc == 2 ? (ul & 1) : 0;
            const uint32_t aph = (uint32_t)(p.nacc == 2 ? (ul >> 1) : ul) & 1u;
            mbar_wait_k<kPair>(&tempty[buf], aph ^ 1);
            tc_fence_after();
            const uint32_t d = tmem_base + (uint32_t)(buf * p.acc_stride);
            for (int kb = w.kb0; kb < w.kb1; ++kb, r.next(S)) {
                const int s = r.s;
                mbar_wait_k<kPair>(&split[s], r.ph);
                tc_fence_after();
                const uint64_t bh = bdesc0 + (uint64_t)s * sstep;
                // A slot: hi at +0..BK-1, lo at +BK..2BK-1
                const uint32_t ah = tmem_base + acol0 + kASlotCols * (uint32_t)s;
                auto mma = [&](uint32_t a_t, uint64_t b_d, uint32_t acc) {
                    if (kPair) tc_mma_tf32_ts_pair_e(d, a_t, b_d, p.idesc, acc);
                    else tc_mma_tf32_ts_e(d, a_t, b_d, p.idesc, acc);
                };
#pragma unroll
                for (int j = 0; j < kKSteps; ++j) {
                    const uint32_t acc = (kb > w.kb0 || j > 0) ? 1u : 0u;
                    const uint32_t a_hi = ah + 8u * j, a_lo = a_hi + BK;
                    const uint64_t b_hi = bh + (uint64_t)j * jstep;
                    mma(a_lo, b_hi, acc);          // a_lo b_hi
                    mma(a_hi, b_hi + lostep, 1u);  // a_hi b_lo
                    mma(a_hi, b_hi, 1u);           // a_hi b_hi
                }
                // frees the smem stage and the TMEM A slot (in both CTAs)
                if (kPair) tc_commit_pair_e(&empty[s]);
                else tc_commit_e(&empty[s]);
            }
            if (kPair) tc_commit_pair_e(&tfull[buf]);
            else tc_commit_e(&tfull[buf]);
        }
    } else if (kPair && warp == kWarpMma) {
        // peer CTA: forward "stage s split done" to the leader's split[s]
        Ring r;
        for (int u = ustart; u < units; u += ustride) {
            Work w = unit_of(p, u);
            for (int kb = w.kb0; kb < w.kb1; ++kb, r.next(S)) {
                mbar_wait(&split[r.s], r.ph);
                mbar_arrive_cluster_e(split_cl0 + 8u * (uint32_t)r.s);
            }
        }
    } else if (warp >= kWarpAx && warp < kWarpBx) {
        // A split: thread = tile row (TMEM lane); TMEM lane quadrant = warp % 4
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const uint32_t tlane = (uint32_t)(q * 32) << 16;
        Ring r;
        for (int u = ustart; u < units; u += ustride) {
            Work w = unit_of(p, u);
            for (int kb = w.kb0; kb < w.kb1; ++kb, r.next(S)) {
                const int s = r.s;
                mbar_wait(&full[s], r.ph);
                const uint32_t a0 = smem0 + (uint32_t)s * p.stage_bytes;
                uint32_t hi[BK], lo[BK];
                if (p.a_kmajor) {
                    // SWIZZLE_128B: 16-B chunk c of row r sits at r*128 + 16*(c ^ (r & 7));
                    // conflict-free across a warp
                    const uint32_t rb = a0 + (uint32_t)row * 128u;
                    const uint32_t sw = (uint32_t)row & 7u;
#pragma unroll
                    for (int c = 0; c < BK / 4; ++c) {
                        const uint4 v = lds128(rb + 16u * ((uint32_t)c ^ sw));
                        hi[4 * c + 0] = v.x; hi[4 * c + 1] = v.y;
                        hi[4 * c + 2] = v.z; hi[4 * c + 3] = v.w;
                    }
                } else {
                    // unswizzled MN-major chunks [m/32][k][32]: lanes read 128 contiguous B
                    const uint32_t cb = a0 + (uint32_t)q * kMnChunkBytes + (uint32_t)lane * 4u;
#pragma unroll
                    for (int k = 0; k < BK; ++k) hi[k] = lds32(cb + 128u * k);
                }
                const uint32_t ta = tmem_base + tlane + acol0 + kASlotCols * (uint32_t)s;
                tmem_st16(ta, hi);
                tmem_st16(ta + 16, hi + 16);
#pragma unroll
                for (int k = 0; k < BK; ++k) lo[k] = tf32_lo(hi[k]);
                tmem_st16(ta + BK, lo);
                tmem_st16(ta + BK + 16, lo + 16);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                mbar_arrive_e(&split[s]);
            }
        }
    } else if (warp >= kWarpBx && warp < kWarpEpi) {
        // B split: b_lo beside the raw B tile
        const int t = threadIdx.x - kWarpBx * 32;
        const uint32_t nB = p.b_bytes / 16;
        Ring r;
        for (int u = ustart; u < units; u += ustride) {
            Work w = unit_of(p, u);
            for (int kb = w.kb0; kb < w.kb1; ++kb, r.next(S)) {
                const int s = r.s;
                mbar_wait(&full[s], r.ph);
                const uint32_t b0 = smem0 + (uint32_t)s * p.stage_bytes + p.a_bytes;
                // 4 loads in flight before the stores (the asm loads/stores
                // are not reordered by the compiler)
                for (uint32_t i0 = t; i0 < nB; i0 += 4 * 128) {
                    uint4 v[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t i = i0 + 128u * k;
                        if (i < nB) v[k] = lds128(b0 + 16u * i);
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t i = i0 + 128u * k;
                        if (i < nB)
                            sts128(b0 + p.b_bytes + 16u * i,
                                   make_uint4(tf32_lo(v[k].x), tf32_lo(v[k].y), tf32_lo(v[k].z),
                                              tf32_lo(v[k].w)));
                    }
                }
                fence_proxy_async();
                __syncwarp();
                mbar_arrive_e(&split[s]);
            }
        }
    } else if (warp >= kWarpEpi) {
        const int q = warp & 3;  // TMEM lane quadrant this warp may access
        int ul = 0;
        for (int u = ustart; u < units; u += ustride, ++ul) {
            Work w = unit_of(p, u);
            const int buf = p.nacc == 2 ? (ul & 1) : 0;
            const uint32_t aph = (uint32_t)(p.nacc == 2 ? (ul >> 1) : ul) & 1u;
            mbar_wait_k<kPair>(&tfull[buf], aph);
            tc_fence_after();
            const int row = w.tm * kRowsPerUnit + (int)rank * BM + q * 32 + lane;
            const uint32_t tbase =
                tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * p.acc_stride);
            for (int c0 = 0; c0 < p.bn; c0 += 16) {
                float v[16];
                tmem_ld16(tbase + c0, v);
                const int col0 = w.tn * p.bn + c0;
                if (row >= p.M || col0 >= p.N) continue;
                if (p.splits > 1) {
                    float* dst = p.ws + ((size_t)w.ks * p.M + row) * p.N + col0;
                    const int lim = min(16, p.N - col0);
                    for (int i = 0; i < lim; ++i) dst[i] = v[i];
                } else {
                    float* dst = p.C + (size_t)row * p.ldc + col0;
                    const int lim = min(16, p.N - col0);
                    const bool vec = lim == 16 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
                    if (vec) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4) {
                            float4 o;
                            if (p.beta != 0.f) {
                                float4 c = *reinterpret_cast<float4*>(dst + i);
                                o = make_float4(p.alpha * v[i] + p.beta * c.x,
                                                p.alpha * v[i + 1] + p.beta * c.y,
                                                p.alpha * v[i + 2] + p.beta * c.z,
                                                p.alpha * v[i + 3] + p.beta * c.w);
                            } else {
                                o = make_float4(p.alpha * v[i], p.alpha * v[i + 1],
                                                p.alpha * v[i + 2], p.alpha * v[i + 3]);
                            }
                            *reinterpret_cast<float4*>(dst + i) = o;
                        }
                    } else {
                        for (int i = 0; i < lim; ++i)
                            dst[i] = p.beta != 0.f ? p.alpha * v[i] + p.beta * dst[i]
                                                   : p.alpha * v[i];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (kPair) mbar_arrive_cluster_e(tempty_cl0 + 8u * (uint32_t)buf);
            else mbar_arrive_e(&tempty[buf]);
        }
    }
    tc_fence_before();
    if (kPair) cluster_sync_all();
    else __syncthreads();
    if (warp == kWarpMma) {
        tc_fence_after();
        if (kPair)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(kTmemCols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(kTmemCols));
    }
}

__global__ void tc_splitk_reduce(const float* __restrict__ ws, int splits, int64_t M, int64_t N,
                                 float alpha, float beta, float* __restrict__ C, int64_t ldc) {
    const int64_t total = M * N;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int z = 0; z < splits; ++z) s += ws[(int64_t)z * total + t];
        int64_t i = t / N, j = t - i * N;
        float* c = C + i * ldc + j;
        *c = beta == 0.f ? alpha * s : alpha * s + beta * *c;
    }
}

// ----------------------------------------------------------------- host ----
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
int g_tc_state = -1;  // -1 unknown, 0 unavailable, 1 available
int g_sms = 148;

bool init_tc() {
    if (g_tc_state >= 0) return g_tc_state == 1;
    g_tc_state = 0;
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (major != 10 || minor != 0) return false;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
        return false;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    g_tc_state = 1;
    return true;
}

// 2-D fp32 map over a row-major [rows x cols] matrix with leading dim ld.
bool encode_2d(CUtensorMap* map, const float* base, uint64_t cols, uint64_t rows, uint64_t ld,
               uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz) {
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * sizeof(float)};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// 3-D view of a row-major [rows x cols] MN-major operand as
// {32 elements, rows, cols/32 chunks} so one box {32, BK, nchunk} lands in smem
// as [chunk][k-row][32] (with swz = SWIZZLE_128B_ATOM_32B: the UMMA
// SWIZZLE_128B_BASE32B layout B needs; unswizzled for A, which the split warps
// read row-per-lane).  Needs ld % 32 == 0 (chunks never cross a row) -- see
// _ops.empty2d.
bool encode_mn3d(CUtensorMap* map, const float* base, uint64_t cols, uint64_t rows, uint64_t ld,
                 uint32_t nchunk, CUtensorMapSwizzle swz) {
    cuuint64_t dims[3] = {32, rows, cdiv(cols, 32)};
    cuuint64_t strides[2] = {ld * sizeof(float), 32 * sizeof(float)};
    cuuint32_t box[3] = {32, (cuuint32_t)BK, nchunk};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims,
                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

struct Plan {
    int bn, tiles_m, tiles_n, splits, num_kb, kb_per_split, stages, acc_stride, nacc;
    uint32_t a_bytes, b_bytes, stage_bytes;
    size_t smem;
};

// pair: CTA-pair plan (256-row units, each CTA loads half of the B tile)
Plan plan_for(int64_t M, int64_t N, int64_t K, int64_t ws_cap_elems, bool b_mn, bool b_mn3d,
              bool pair) {
    Plan pl;
    pl.tiles_n = (int)cdiv(N, kMaxBn);
    // MN-major B is addressed in whole 32-column chunks (per CTA half when paired)
    const int gran = b_mn ? (pair ? 64 : (b_mn3d ? 32 : 16)) : (pair ? 32 : 16);
    pl.bn = (int)(cdiv(cdiv(N, pl.tiles_n), gran) * gran);
    pl.tiles_m = (int)cdiv(M, pair ? 2 * BM : BM);
    pl.num_kb = (int)cdiv(K, BK);
    const int slots_machine = pair ? g_sms / 2 : g_sms;
    int64_t base = (int64_t)pl.tiles_m * pl.tiles_n;
    int splits = 1;
    if (base < 4 * slots_machine) {
        double best = 0;
        int maxs = (int)std::max<int64_t>(1, pl.num_kb / 8);
        for (int s = 1; s <= std::min(64, maxs); ++s) {
            int64_t units = base * s;
            if (s > 1 && (int64_t)s * M * N > ws_cap_elems) break;
            double waves = (double)cdiv(units, slots_machine);
            double eff = (double)units / (waves * slots_machine);
            // prefer enough units to fill the machine, then balanced waves
            double score = std::min(1.0, (double)units / slots_machine) * eff;
            if (score > best + 0.02) { best = score; splits = s; }
        }
    }
    // The tensor core's fp32 accumulation error grows ~linearly with the
    // chain length (measured: 1.8e-4 relative at K = 262144), so K is cut
    // into chains of at most 32768 -- split-K partials summed in fp32 by the
    // reduce pass (workspace permitting).
    const int max_kb = 32768 / BK;
    if (cdiv(pl.num_kb, splits) > max_kb) {
        const int s2 = (int)cdiv(pl.num_kb, max_kb);
        if ((int64_t)s2 * M * N <= ws_cap_elems) splits = std::max(splits, s2);
    }
    pl.kb_per_split = (int)cdiv(pl.num_kb, splits);
    pl.splits = (int)cdiv(pl.num_kb, pl.kb_per_split);
    pl.a_bytes = BM * BK * 4;
    // B columns held per CTA; MN-major B is loaded in 32-wide chunks (a partial
    // last chunk is padded)
    const int bcols = pair ? pl.bn / 2 : pl.bn;
    pl.b_bytes = b_mn ? (uint32_t)cdiv(bcols, 32) * kMnChunkBytes : (uint32_t)bcols * BK * 4;
    pl.stage_bytes = pl.a_bytes + 2 * pl.b_bytes;
    // TMEM: two accumulator buffers, then one 32-column A slot per stage
    pl.acc_stride = (int)cdiv(pl.bn, 32) * 32;
    // double-buffer the accumulator (epilogue overlaps the next tile) only when
    // that still leaves room for 4 A slots
    pl.nacc = ((int)kTmemCols - 2 * pl.acc_stride) / (int)kASlotCols >= 4 ? 2 : 1;
    const int slots = ((int)kTmemCols - pl.nacc * pl.acc_stride) / (int)kASlotCols;
    const size_t budget = 220 * 1024;
    int st = (int)((budget - 1024 - 256) / pl.stage_bytes);
    pl.stages = std::max(2, std::min({kMaxStages, st, slots}));
    pl.smem = 1024 + (size_t)pl.stages * pl.stage_bytes + (3 * pl.stages + 4) * 8 + 16;
    return pl;
}

// CTA pairs pay off once there are enough 256-row units to fill the machine
bool use_pair(int64_t M) {
    return M > BM;
}

}  // namespace

bool tc_available() { return init_tc(); }

int64_t gemm_tc_ws_bytes(int ta, int tb, int64_t M, int64_t N, int64_t K) {
    (void)ta;
    (void)tb;
    if (!init_tc()) return 0;
    Plan pl = plan_for(M, N, K, INT64_MAX, tb == 0, false, use_pair(M));
    return pl.splits > 1 ? (int64_t)pl.splits * M * N * 4 : 0;
}

int gemm_tc_3xtf32(int ta, int tb, int64_t M, int64_t N, int64_t K, float alpha, const float* A,
                   int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc,
                   void* ws, int64_t ws_bytes, cudaStream_t st) {
    if (!init_tc()) return SKP_ERR_UNSUPPORTED;
    if (M == 0 || N == 0) return SKP_OK;
    if (K == 0 || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return SKP_ERR_UNSUPPORTED;
    // TMA: 16-B aligned bases and row strides
    if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15) ||
        (lda & 3) || (ldb & 3)) {
        set_error("unsupported: 3xTF32 tcgen05 path needs 16-byte aligned operands and leading "
                  "dimensions (lda=%lld ldb=%lld)", (long long)lda, (long long)ldb);
        return SKP_ERR_UNSUPPORTED;
    }
    const int64_t cap = ws ? ws_bytes / 4 : 0;
    // one 3-D box per MN-major operand per stage when rows are 128-byte padded
    const bool a_mn3d = ta && (lda % 32 == 0);
    const bool b_mn3d = !tb && (ldb % 32 == 0);
    const bool pair = use_pair(M);
    Plan pl = plan_for(M, N, K, cap, tb == 0, b_mn3d, pair);
    if (pl.splits > 1 && (!ws || (int64_t)pl.splits * M * N * 4 > ws_bytes)) {
        pl = plan_for(M, N, K, 0, tb == 0, b_mn3d, pair);  // no split-K without workspace
    }
    TcParams p;
    p.M = (int)M; p.N = (int)N; p.K = (int)K;
    p.bn = pl.bn; p.tiles_m = pl.tiles_m; p.tiles_n = pl.tiles_n; p.splits = pl.splits;
    p.kb_per_split = pl.kb_per_split; p.num_kb = pl.num_kb;
    p.a_kmajor = ta ? 0 : 1;   // op(A) = A (M x K, K contiguous) or A^T (A is K x M)
    p.b_kmajor = tb ? 1 : 0;   // op(B) = B (K x N, N contiguous) or B^T (B is N x K)
    p.alpha = alpha; p.beta = beta; p.C = C; p.ldc = ldc;
    p.ws = pl.splits > 1 ? reinterpret_cast<float*>(ws) : nullptr;
    p.stages = pl.stages; p.a_bytes = pl.a_bytes; p.b_bytes = pl.b_bytes;
    p.stage_bytes = pl.stage_bytes;
    p.acc_stride = pl.acc_stride;
    p.nacc = pl.nacc;
    // A comes from TMEM (always K-major there); B's major-ness from its layout
    p.idesc = (1u << 4) | (2u << 7) | (2u << 10) |
              ((uint32_t)(!p.b_kmajor) << 16) | ((uint32_t)(p.bn >> 3) << 17) |
              ((uint32_t)((pair ? 2 * BM : BM) >> 4) << 24);
    CUtensorMap ma, mb;
    const CUtensorMapSwizzle kSw = CU_TENSOR_MAP_SWIZZLE_128B, mSw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    p.a_mn3d = a_mn3d;
    p.b_mn3d = b_mn3d;
    bool ok;
    if (p.a_kmajor) ok = encode_2d(&ma, A, (uint64_t)K, (uint64_t)M, lda, BK, BM, kSw);
    else if (p.a_mn3d)
        ok = encode_mn3d(&ma, A, (uint64_t)M, (uint64_t)K, lda, BM / 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    else ok = encode_2d(&ma, A, (uint64_t)M, (uint64_t)K, lda, 32, BK, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!ok) {
    }
    const int bcols = pair ? p.bn / 2 : p.bn;  // B columns loaded per CTA
    if (!ok) {
    } else if (p.b_kmajor) ok = encode_2d(&mb, B, (uint64_t)K, (uint64_t)N, ldb, BK, (uint32_t)bcols, kSw);
    else if (p.b_mn3d) ok = encode_mn3d(&mb, B, (uint64_t)N, (uint64_t)K, ldb, (uint32_t)cdiv(bcols, 32), mSw);
    else ok = encode_2d(&mb, B, (uint64_t)N, (uint64_t)K, ldb, 32, BK, mSw);
    if (!ok) {
        set_error("cuTensorMapEncodeTiled failed");
        return SKP_ERR_UNSUPPORTED;
    }
    const int units = p.tiles_m * p.tiles_n * p.splits;
    int grid;
    if (pair) {
        SKP_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
        grid = 2 * std::min(units, g_sms / 2);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = pl.smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        SKP_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<true>, ma, mb, p));
        SKP_LAUNCHED(gemm_tc_kernel_pair);
    } else {
        SKP_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
        grid = std::min(units, g_sms);
        gemm_tc_kernel<false><<<grid, kThreads, pl.smem, st>>>(ma, mb, p);
        SKP_LAUNCHED(gemm_tc_kernel);
    }
    if (p.splits > 1) {
        int64_t blocks = std::min<int64_t>(cdiv(M * N, 256), (int64_t)g_sms * 8);
        tc_splitk_reduce<<<(unsigned)blocks, 256, 0, st>>>(p.ws, p.splits, M, N, alpha, beta, C,
                                                           ldc);
        SKP_LAUNCHED(tc_splitk_reduce);
    }
    return SKP_OK;
}

}  // namespace skp
