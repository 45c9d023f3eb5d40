// K4: FP32 GEMM on the sm_100a tensor cores by the 3xTF32 split, tcgen05/TMEM.
//
//   C = alpha * op(A) op(B) + beta * C,   a = a_hi + a_lo,
//   a.b ~= a_hi.b_hi + a_hi.b_lo + a_lo.b_hi   (error ~2^-20 relative per term,
//   below the fp32 accumulation error of the TMEM accumulator for K >~ 100)
// kind::tf32 reads fp32 containers and TRUNCATES to the TF32 grid (measured on
// B200: raw-operand products match truncated inputs to accumulation noise and
// miss round-to-nearest by ~500x), so the raw tile IS a_hi and only
// a_lo = a - trunc(a) (exact in fp32) is materialised beside it.
//
// One persistent CTA per SM, warp-specialised (10 warps):
//   warp 0      TMA producer: raw fp32 tiles -> smem ring (SWIZZLE_64B, BK=16)
//   warp 1      MMA issuer: one elected lane issues 6 tcgen05.mma.kind::tf32 per
//               stage (2 K-steps x 3 products) into a TMEM accumulator; owns the
//               TMEM allocation (2 x 256 columns = double-buffered accumulators)
//   warps 2-9   split: lo = x - trunc_tf32(x) beside each raw tile
//   warps 10-13 epilogue: tcgen05.ld 32x32b -> alpha/beta -> global (or split-K
//               partials), overlapping the next tile's main loop
// Operands may be K-major (K contiguous, one 2-D TMA box per tile) or MN-major
// (MN contiguous, one 16-wide box per 16 MN elements); the UMMA descriptors
// carry the major-ness, so no transposes are ever materialised.
// Tiles: BM = 128 (UMMA M), BN = runtime multiple of 16 <= 256, BK = 16.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <stdlib.h>

#include "common.cuh"
#include "gemm.h"

namespace skp {
namespace {

constexpr int BM = 128;
constexpr int BK = 16;
constexpr int kWarpTma = 0, kWarpMma = 1, kWarpXf = 2, kNumXf = 8, kWarpEpi = 10, kNumEpi = 4;
constexpr int kThreads = 32 * (kWarpEpi + kNumEpi);
constexpr uint32_t kTmemCols = 512;
constexpr int kMaxStages = 8;

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
    int xf_mode;  // 0: 3xTF32 (split in smem); 1: debug -- raw operands, one product
};

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    long long t0 = 0;
    for (int it = 0;; ++it) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
        if (ok) return;
        // watchdog: a protocol bug becomes a trap (error), never a hung GPU
        if (it == 64) t0 = clock64();
        if (it > 64 && (it & 1023) == 0 && clock64() - t0 > (long long)40e9) __trap();
    }
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// Round-to-nearest (ties away) onto the TF32 grid: 2 integer ops (cvt.rna.tf32
// is emulated by ~10 instructions on sm_100).
__device__ __forceinline__ uint32_t tf32_round_bits(uint32_t u) {
    return (u + 0x1000u) & 0xFFFFE000u;
}
// lo = x - trunc_tf32(x): exact in fp32; the tensor core truncates it again.
__device__ __forceinline__ uint32_t tf32_lo(uint32_t x) {
    return __float_as_uint(__uint_as_float(x) - __uint_as_float(x & 0xFFFFE000u));
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// UMMA shared-memory descriptors (sm_100, version 1).
//  K-major : SWIZZLE_64B, rows of 64 B (16 fp32 of K), 8-row atoms (SBO 512 B);
//            K-step of 8 = +32 B inside the atom.
//  MN-major: SWIZZLE_128B_BASE32B -- the only MN-major layout tf32 accepts:
//            atoms of 32 MN-elements (128 B) x 4 K-rows, 32-B chunks swizzled
//            (TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B); LBO = MN-chunk stride
//            (BK rows x 128 B), SBO = 4-row atom stride (512 B); K-step of 8 =
//            +1 KB.
constexpr uint32_t kLayoutSW64 = 4, kLayoutSW128Base32B = 1;
constexpr uint32_t kMnChunkBytes = 32 * BK * 4;  // one TMA box: 32 MN x BK K

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version for tcgen05
    d |= (uint64_t)layout << 61;
    return d;
}
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int kmajor, int j) {
    return kmajor ? make_desc(base + 32u * j, 16u, 512u, kLayoutSW64)
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

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&split[s], kNumXf);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kNumEpi);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kWarpMma) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto stage_a = [&](int s) { return smem + (size_t)s * p.stage_bytes; };
    auto stage_alo = [&](int s) { return stage_a(s) + p.a_bytes; };
    auto stage_b = [&](int s) { return stage_a(s) + 2 * p.a_bytes; };
    auto stage_blo = [&](int s) { return stage_b(s) + p.b_bytes; };

    if (warp == kWarpTma) {
        if (lane == 0) {
            int it = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                Work w = unit_of(p, u);
                const int m0 = w.tm * BM, n0 = w.tn * p.bn;
                for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                    const int s = it % S;
                    const uint32_t ph = (it / S) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_expect_tx(&full[s], p.a_bytes + p.b_bytes);
                    const int k0 = kb * BK;
                    if (p.a_kmajor) {
                        tma_load_2d(&map_a, &full[s], stage_a(s), k0, m0);
                    } else {
                        for (int c = 0; c < BM / 32; ++c)
                            tma_load_2d(&map_a, &full[s], stage_a(s) + c * kMnChunkBytes,
                                        m0 + 32 * c, k0);
                    }
                    if (p.b_kmajor) {
                        tma_load_2d(&map_b, &full[s], stage_b(s), k0, n0);
                    } else {
                        for (int c = 0; c < (p.bn + 31) / 32; ++c)
                            tma_load_2d(&map_b, &full[s], stage_b(s) + c * kMnChunkBytes,
                                        n0 + 32 * c, k0);
                    }
                }
            }
        }
    } else if (warp == kWarpMma) {
        int it = 0, ul = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++ul) {
            Work w = unit_of(p, u);
            const int buf = ul & 1;
            const uint32_t aph = (ul >> 1) & 1;
            mbar_wait(&tempty[buf], aph ^ 1);
            tc_fence_after();
            const uint32_t d = tmem_base + (uint32_t)(buf * 256);
            for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                const int s = it % S;
                const uint32_t ph = (it / S) & 1;
                mbar_wait(&split[s], ph);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t ah = smem_u32(stage_a(s)), al = smem_u32(stage_alo(s));
                    const uint32_t bh = smem_u32(stage_b(s)), bl = smem_u32(stage_blo(s));
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const uint64_t dah = operand_desc(ah, p.a_kmajor, j);
                        const uint64_t dal = operand_desc(al, p.a_kmajor, j);
                        const uint64_t dbh = operand_desc(bh, p.b_kmajor, j);
                        const uint64_t dbl = operand_desc(bl, p.b_kmajor, j);
                        const uint32_t acc = (kb > w.kb0 || j > 0) ? 1u : 0u;
                        if (p.xf_mode == 1) {
                            tc_mma_tf32(d, dah, dbh, p.idesc, acc);
                            continue;
                        }
                        tc_mma_tf32(d, dal, dbh, p.idesc, acc);
                        tc_mma_tf32(d, dah, dbl, p.idesc, 1u);
                        tc_mma_tf32(d, dah, dbh, p.idesc, 1u);
                    }
                    tc_commit(&empty[s]);
                }
                __syncwarp();
            }
            if (lane == 0) tc_commit(&tfull[buf]);
            __syncwarp();
        }
    } else if (warp >= kWarpXf && warp < kWarpXf + kNumXf) {
        const int t = threadIdx.x - kWarpXf * 32;
        int it = 0;
        const uint32_t nA = p.a_bytes / 16, nB = p.b_bytes / 16;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            Work w = unit_of(p, u);
            for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                const int s = it % S;
                const uint32_t ph = (it / S) & 1;
                mbar_wait(&full[s], ph);
                if (p.xf_mode == 1) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&split[s]);
                    continue;
                }
                // layout per stage: [A_hi | A_lo | B_hi | B_lo]; lo sits one buffer
                // past its hi, so each 16-B granule maps to (src, src + bytes)
                const uint32_t a0 = smem_u32(stage_a(s)), b0 = smem_u32(stage_b(s));
                for (uint32_t i = t; i < nA + nB; i += kNumXf * 32) {
                    const bool isa = i < nA;
                    const uint32_t src = isa ? a0 + 16u * i : b0 + 16u * (i - nA);
                    const uint32_t dlo = src + (isa ? p.a_bytes : p.b_bytes);
                    const uint4 v = lds128(src);
                    sts128(dlo, make_uint4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w)));
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(&split[s]);
            }
        }
    } else if (warp >= kWarpEpi) {
        const int q = warp & 3;  // TMEM lane quadrant this warp may access
        int ul = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++ul) {
            Work w = unit_of(p, u);
            const int buf = ul & 1;
            const uint32_t aph = (ul >> 1) & 1;
            mbar_wait(&tfull[buf], aph);
            tc_fence_after();
            const int row = w.tm * BM + q * 32 + lane;
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * 256);
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
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kWarpMma) {
        tc_fence_after();
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
    if (getenv("SKP_DISABLE_TCGEN05")) return false;
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

struct Plan {
    int bn, tiles_m, tiles_n, splits, num_kb, kb_per_split, stages;
    uint32_t a_bytes, b_bytes, stage_bytes;
    size_t smem;
};

Plan plan_for(int64_t M, int64_t N, int64_t K, int64_t ws_cap_elems, bool b_mn) {
    Plan pl;
    pl.tiles_n = (int)cdiv(N, 256);
    pl.bn = (int)(cdiv(cdiv(N, pl.tiles_n), 16) * 16);
    pl.tiles_m = (int)cdiv(M, BM);
    pl.num_kb = (int)cdiv(K, BK);
    int64_t base = (int64_t)pl.tiles_m * pl.tiles_n;
    int splits = 1;
    if (base < 4 * g_sms) {
        double best = 0;
        int maxs = (int)std::max<int64_t>(1, pl.num_kb / 8);
        for (int s = 1; s <= std::min(64, maxs); ++s) {
            int64_t units = base * s;
            if (s > 1 && (int64_t)s * M * N > ws_cap_elems) break;
            double waves = (double)cdiv(units, g_sms);
            double eff = (double)units / (waves * g_sms);
            // prefer enough units to fill the machine, then balanced waves
            double score = std::min(1.0, (double)units / g_sms) * eff;
            if (score > best + 0.02) { best = score; splits = s; }
        }
    }
    pl.kb_per_split = (int)cdiv(pl.num_kb, splits);
    pl.splits = (int)cdiv(pl.num_kb, pl.kb_per_split);
    pl.a_bytes = BM * BK * 4;
    // MN-major B is loaded in 32-wide chunks (a partial last chunk is padded)
    pl.b_bytes = b_mn ? (uint32_t)cdiv(pl.bn, 32) * kMnChunkBytes : (uint32_t)pl.bn * BK * 4;
    pl.stage_bytes = 2 * pl.a_bytes + 2 * pl.b_bytes;
    const size_t budget = 220 * 1024;
    int st = (int)((budget - 1024 - 256) / pl.stage_bytes);
    pl.stages = std::max(2, std::min(kMaxStages, st));
    pl.smem = 1024 + (size_t)pl.stages * pl.stage_bytes + (3 * pl.stages + 4) * 8 + 16;
    return pl;
}

}  // namespace

bool tc_available() { return init_tc(); }

int64_t gemm_tc_ws_bytes(int ta, int tb, int64_t M, int64_t N, int64_t K) {
    (void)ta;
    (void)tb;
    if (!init_tc()) return 0;
    Plan pl = plan_for(M, N, K, INT64_MAX, tb == 0);
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
    Plan pl = plan_for(M, N, K, cap, tb == 0);
    if (pl.splits > 1 && (!ws || (int64_t)pl.splits * M * N * 4 > ws_bytes)) {
        pl = plan_for(M, N, K, 0, tb == 0);  // no split-K without workspace
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
    p.xf_mode = getenv("SKP_TC_RAW1") ? 1 : 0;
    p.idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(!p.a_kmajor) << 15) |
              ((uint32_t)(!p.b_kmajor) << 16) | ((uint32_t)(p.bn >> 3) << 17) |
              ((uint32_t)(BM >> 4) << 24);
    CUtensorMap ma, mb;
    const CUtensorMapSwizzle kSw = CU_TENSOR_MAP_SWIZZLE_64B, mSw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    bool ok = p.a_kmajor ? encode_2d(&ma, A, (uint64_t)K, (uint64_t)M, lda, BK, BM, kSw)
                         : encode_2d(&ma, A, (uint64_t)M, (uint64_t)K, lda, 32, BK, mSw);
    ok = ok && (p.b_kmajor ? encode_2d(&mb, B, (uint64_t)K, (uint64_t)N, ldb, BK, (uint32_t)p.bn, kSw)
                           : encode_2d(&mb, B, (uint64_t)N, (uint64_t)K, ldb, 32, BK, mSw));
    if (!ok) {
        set_error("cuTensorMapEncodeTiled failed");
        return SKP_ERR_UNSUPPORTED;
    }
    SKP_CUDA(cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)pl.smem));
    const int units = p.tiles_m * p.tiles_n * p.splits;
    const int grid = std::min(units, g_sms);
    gemm_tc_kernel<<<grid, kThreads, pl.smem, st>>>(ma, mb, p);
    SKP_LAUNCHED(gemm_tc_kernel);
    if (p.splits > 1) {
        int64_t blocks = std::min<int64_t>(cdiv(M * N, 256), (int64_t)g_sms * 8);
        tc_splitk_reduce<<<(unsigned)blocks, 256, 0, st>>>(p.ws, p.splits, M, N, alpha, beta, C,
                                                           ldc);
        SKP_LAUNCHED(tc_splitk_reduce);
    }
    return SKP_OK;
}

}  // namespace skp
