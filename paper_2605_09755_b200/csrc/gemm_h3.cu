// K4h: FP32 GEMM from PRE-SPLIT fp16 operands on the sm_100a tensor cores
// ("3xFP16"), tcgen05.mma.kind::f16 with fp32 accumulation in TMEM.
//
//   x * 2^e = x_hi + x_lo + O(2^-22 |x| 2^e),   x_hi = fp16(x 2^e),
//   x_lo = fp16(x 2^e - x_hi),  e = 15 - ceil(log2 max|X|)  (one power of two
//   per matrix, so max|x| 2^e lies in [2^14, 2^15): no fp16 overflow, and the
//   bulk of the entries far above the fp16 subnormal range)
//   a.b ~= 2^-(ea+eb) (a_lo b_hi + a_hi b_lo + a_hi b_hi)
//
// Why: 3xTF32 (gemm_tc.cu) already runs the TF32 tensor pipe at ~93% of its
// peak; the only way past it is a faster pipe.  kind::f16 runs at twice the
// TF32 rate, and an 11+11-bit fp16 pair carries the same 22 significant bits
// as a TF32 hi/lo pair (fp16's narrow exponent range is what the per-matrix
// power-of-two scale handles).  Per-product error 2^-22 vs 3xTF32's 2^-20.
//
// The operands are split ONCE per matrix in HBM (skp_split_h2_f32: hi and lo
// planes of 2 bytes each = the fp32 footprint), not per tile: A~ (m x l) is
// reused by all 1+2q power-iteration products, and with no split warps the
// kernel is a plain TMA -> MMA -> epilogue pipeline whose shared-memory traffic
// (TMA writes + operand reads) stays under the 128 B/clk the split version
// would have exceeded at the f16 rate.
//
// One persistent CTA (or CTA pair) per SM, warp-specialised (6 warps):
//   warp 0     TMA producer: A_hi, A_lo, B_hi, B_lo tiles -> smem ring
//   warp 1     MMA issuer (leader CTA): 12 tcgen05.mma per stage (4 K-steps of
//              16 x 3 products), both operands from shared memory
//   warps 2-5  epilogue: tcgen05.ld -> 2^-(ea+eb) alpha (+ beta C) -> global
// Operand layouts: A K-major (op(A) = A, M x K, K contiguous) or MN-major
// (op(A) = A^T, A stored K x M) -- SWIZZLE_128B, 64 fp16 per 128-byte row;
// B always K-major (stored N x K; the split kernel transposes small B's for
// free).  CTA pair (cta_group::2, M = 256): each CTA loads its own 128 A rows
// and half of the B tile, both CTAs' TMA signal the leader's full barrier.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <stdlib.h>
#include <stdio.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace skp {
namespace {

constexpr int HM = 128;          // UMMA M per CTA
constexpr int HK = 64;           // fp16 K per stage: one 128-byte swizzled row
constexpr int kHKSteps = HK / 16;  // f16 UMMA K = 16
constexpr int kHWarpTma = 0, kHWarpMma = 1, kHWarpEpi = 2, kHNumEpi = 12;
// 16-column groups per epilogue thread: the accumulator lives in registers
// across the chunks of a unit, 3 column thirds x 4 groups -> bn <= 192 (14
// warps leave 128 registers a thread: 4 warps share an SMSP's 16K registers)
constexpr int kHEpiCols = 4;
constexpr int kHEpiParts = kHNumEpi / 4;
constexpr int kHMaxBn = kHEpiParts * 16 * kHEpiCols;
constexpr int kHThreads = 32 * (kHWarpEpi + kHNumEpi);
constexpr uint32_t kHTmemCols = 512;
constexpr int kHMaxStages = 8;
constexpr uint32_t kHChunkBytes = 64 * HK * 2;  // MN-major A: 64 M x HK K per TMA box chunk

struct H3Params {
    int M, N, K;
    int bn, tiles_m, tiles_n, splits, kb_per_split, num_kb;
    int a_kmajor;
    int b_kmajor;  // 0: B stored K x N (N contiguous; the SYRK's second operand)
    int sym;       // > 0: C = A^T A, units = the lower-triangle tiles x splits (mirrored after)
    int sym_tiles; // lower-triangle tiles (sym)
    int tri_k;     // 1: B (stored N x K) is lower triangular: N tile tn needs K < (tn + 1) bn
    unsigned* prog;  // pacing slots (one per CTA; see h_pace), or null
    int pace;        // > 0: a producer stays within pace K blocks of the slowest CTA of its wave
    float alpha, beta;
    float* C;
    long long ldc;
    float* ws;
    int stages;
    uint32_t a_bytes, b_bytes, stage_bytes;
    uint32_t idesc;
    int acc_stride;
    const int* a_e;
    const int* b_e;
    int chunk_kb;  // K blocks per accumulation chunk (promotion period)
    int b_lo;      // 1: 3 products; 0: B's lo plane dropped (2 products, B to 11 bits)
    // emit mode (emit_hi != null): instead of C, write the fp16 split of
    // C^T (N x M planes, ld emit_ld) with exponent e_out = emit_fixed ?
    // emit_e_fixed : ea + eb - emit_shift, stored to *emit_e; an entry that
    // does not fit fp16 sets *overflow
    __half* emit_hi;
    __half* emit_lo;
    long long emit_ld;
    int emit_shift, emit_fixed, emit_e_fixed;
    int* emit_e;
    int* overflow;
};

// TMA 2-D / 3-D loads signalling a barrier given by its shared::cluster
// address (the leader CTA's barrier when paired: .cta_group::2 lets the peer's
// copy complete_tx on it)
template <bool kPair>
__device__ __forceinline__ void h_tma_2d(const CUtensorMap* map, uint32_t bar_cl, uint32_t dst,
                                         int c0, int c1) {
    if (kPair)
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
            "@p cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];\n\t}" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cl), "r"(c0), "r"(c1)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
            "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];\n\t}" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cl), "r"(c0), "r"(c1)
            : "memory");
}
template <bool kPair>
__device__ __forceinline__ void h_tma_3d(const CUtensorMap* map, uint32_t bar_cl, uint32_t dst,
                                         int c0, int c1, int c2) {
    if (kPair)
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
            "@p cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5}], [%2];\n\t}" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cl), "r"(c0), "r"(c1), "r"(c2)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
            "@p cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5}], [%2];\n\t}" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cl), "r"(c0), "r"(c1), "r"(c2)
            : "memory");
}
// D[tmem] (+)= A[smem desc] * B[smem desc], kind::f16 (fp16 in, fp32 accumulate)
template <bool kPair>
__device__ __forceinline__ void h_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                      uint32_t acc) {
    if (kPair)
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t.reg .b32 r;\n\t"
            "setp.ne.b32 q, %4, 0;\n\t"
            "elect.sync r|p, 0xffffffff;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t.reg .b32 r;\n\t"
            "setp.ne.b32 q, %4, 0;\n\t"
            "elect.sync r|p, 0xffffffff;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
}

// mbarrier wait for the epilogue warps: back off between polls (12 warps
// spinning on try_wait took issue slots from the TMA / MMA warps)
__device__ __forceinline__ void mbar_wait_idle(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    long long t0 = 0;
    for (int it = 0;; ++it) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(128);
        if (it == 64) t0 = clock64();
        if (it > 64 && (it & 1023) == 0 && clock64() - t0 > (long long)40e9) __trap();
    }
}

// acc[0..15] += v[0..15] as ONE volatile asm: it stays ordered against the
// tcgen05.ld of the next 16 columns, so only 16 loaded values are live at a
// time (left to the compiler, all groups' loads were hoisted and spilled)
__device__ __forceinline__ void acc_add16(float* acc, const float* v) {
    asm volatile(
        "add.f32 %0, %0, %16;\n\tadd.f32 %1, %1, %17;\n\tadd.f32 %2, %2, %18;\n\t"
        "add.f32 %3, %3, %19;\n\tadd.f32 %4, %4, %20;\n\tadd.f32 %5, %5, %21;\n\t"
        "add.f32 %6, %6, %22;\n\tadd.f32 %7, %7, %23;\n\tadd.f32 %8, %8, %24;\n\t"
        "add.f32 %9, %9, %25;\n\tadd.f32 %10, %10, %26;\n\tadd.f32 %11, %11, %27;\n\t"
        "add.f32 %12, %12, %28;\n\tadd.f32 %13, %13, %29;\n\tadd.f32 %14, %14, %30;\n\t"
        "add.f32 %15, %15, %31;"
        : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3]), "+f"(acc[4]), "+f"(acc[5]),
          "+f"(acc[6]), "+f"(acc[7]), "+f"(acc[8]), "+f"(acc[9]), "+f"(acc[10]), "+f"(acc[11]),
          "+f"(acc[12]), "+f"(acc[13]), "+f"(acc[14]), "+f"(acc[15])
        : "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
          "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
          "f"(v[15]));
}

struct HWork {
    int tm, tn, ks, kb0, kb1;
};

// Wave pacing for the long-K products (SYRK G = A~^T A~, B^T = A^T Q): the
// CTAs working on the same wave of units read the same K slice of the shared
// operand (A~ / A) at the same time only while they stay in step -- left
// alone they drift apart by more than the 126 MB L2 holds, and ncu measured
// A read 8x (K4s at C5: 1.06 TB for a 128 GB A).  Each TMA producer publishes
// (wave << 20 | k block) in its slot and, every 4 K blocks, waits while it is
// more than `pace` K blocks ahead of the slowest CTA of its own wave (other
// waves are ignored, so the slowest CTA never waits: no deadlock).
__device__ __forceinline__ unsigned h_ld_slot(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void h_st_slot(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void h_pace(unsigned* prog, int pace, unsigned wave, int kb_rel,
                                       int& lo_cache) {
    const int lane = threadIdx.x & 31;
    const unsigned me = (wave << 20) | (unsigned)kb_rel;
    if (lane == 0) h_st_slot(prog + blockIdx.x, me);
    if (kb_rel == 0) lo_cache = 0;
    // the slots are read only when this CTA may be getting ahead: the ring
    // must not drain while the producer polls
    if (kb_rel - lo_cache <= pace / 2) return;
    for (int it = 0;; ++it) {
        int lo = kb_rel;
        for (int i = lane; i < (int)gridDim.x; i += 32) {
            const unsigned v = h_ld_slot(prog + i);
            if ((v >> 20) == wave) lo = min(lo, (int)(v & 0xFFFFFu));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        lo_cache = lo;
        if (kb_rel - lo <= pace || it > (1 << 22)) return;
        __nanosleep(200);
    }
}
__device__ __forceinline__ void h_pace_done(unsigned* prog) {
    if ((threadIdx.x & 31) == 0) h_st_slot(prog + blockIdx.x, 0xFFFFFFFFu);
}
template <bool kPair>
__device__ __forceinline__ HWork h_unit(const H3Params& p, int u) {
    // N-tiles of one M block are adjacent units: co-resident CTAs share the A
    // row block through L2
    HWork w;
    if (p.sym) {
        // lower triangle only: M block tm needs the N tiles that start at or
        // before its last row (the tiles are enumerated block row by row);
        // split-K slices of one tile are sym_tiles units apart
        constexpr int R = kPair ? 2 * HM : HM;
        const int t = u % p.sym_tiles;
        int tm = 0, base = 0;
        for (;;) {
            const int c = min(p.tiles_n, ((tm + 1) * R + p.bn - 1) / p.bn);
            if (t < base + c) break;
            base += c;
            ++tm;
        }
        w.tm = tm;
        w.tn = t - base;
        w.ks = u / p.sym_tiles;
        w.kb0 = w.ks * p.kb_per_split;
        w.kb1 = min(w.kb0 + p.kb_per_split, p.num_kb);
        return w;
    }
    w.tn = u % p.tiles_n;
    const int r = u / p.tiles_n;
    w.tm = r % p.tiles_m;
    w.ks = r / p.tiles_m;
    w.kb0 = w.ks * p.kb_per_split;
    w.kb1 = min(w.kb0 + p.kb_per_split, p.num_kb);
    if (p.tri_k) w.kb1 = min(w.kb1, ((w.tn + 1) * p.bn + HK - 1) / HK);
    return w;
}

template <bool kPair, int kEC = kHEpiCols>
__global__ void __launch_bounds__(kHThreads, 1)
gemm_h3_kernel(const __grid_constant__ CUtensorMap map_ah, const __grid_constant__ CUtensorMap map_al,
               const __grid_constant__ CUtensorMap map_bh, const __grid_constant__ CUtensorMap map_bl,
               const H3Params p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * p.stage_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* tfull = bars + 2 * S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int units = p.sym ? p.sym : p.tiles_m * p.tiles_n * p.splits;
    const uint32_t rank = kPair ? cluster_rank() : 0u;
    const bool leader = rank == 0;
    const int ustart = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int ustride = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    constexpr int kRowsPerUnit = kPair ? 2 * HM : HM;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);  // the leader's expect_tx arrive (+ tx of both CTAs)
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kPair ? 2 * kHNumEpi : kHNumEpi);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kHWarpMma) {
        if (kPair) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kHTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kHTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    if (kPair) cluster_sync_all();
    else __syncthreads();
    tc_fence_after();
    const uint32_t full_cl0 = kPair ? mapa_shared(smem_u32(full), 0) : smem_u32(full);
    const uint32_t tempty_cl0 = kPair ? mapa_shared(smem_u32(tempty), 0) : 0u;
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t smem0 = smem_u32(smem);

    if (warp == kHWarpTma) {
        Ring r;
        const int bcols = kPair ? p.bn / 2 : p.bn;
        unsigned wave = 0;
        int lo_cache = 0;
        for (int u = ustart; u < units; u += ustride, ++wave) {
            const HWork w = h_unit<kPair>(p, u);
            const int m0 = w.tm * kRowsPerUnit + (int)rank * HM;
            const int n0 = w.tn * p.bn + (int)rank * bcols;
            for (int kb = w.kb0; kb < w.kb1; ++kb, r.next(S)) {
                const int s = r.s;
                if (p.pace && ((kb - w.kb0) & 3) == 0)
                    h_pace(p.prog, p.pace, wave, kb - w.kb0, lo_cache);
                mbar_wait(&empty[s], r.ph ^ 1);
                if (leader) mbar_expect_tx_e(&full[s], (kPair ? 2u : 1u) * p.stage_bytes);
                const uint32_t bar = full_cl0 + 8u * (uint32_t)s;
                const uint32_t st = smem0 + (uint32_t)s * p.stage_bytes;
                const int k0 = kb * HK;
                if (p.a_kmajor) {
                    h_tma_2d<kPair>(&map_ah, bar, st, k0, m0);
                    h_tma_2d<kPair>(&map_al, bar, st + p.a_bytes, k0, m0);
                } else {
                    h_tma_3d<kPair>(&map_ah, bar, st, 0, k0, m0 / 64);
                    h_tma_3d<kPair>(&map_al, bar, st + p.a_bytes, 0, k0, m0 / 64);
                }
                if (p.b_kmajor) {
                    h_tma_2d<kPair>(&map_bh, bar, st + 2 * p.a_bytes, k0, n0);
                    if (p.b_lo)
                        h_tma_2d<kPair>(&map_bl, bar, st + 2 * p.a_bytes + p.b_bytes, k0, n0);
                } else {
                    h_tma_3d<kPair>(&map_bh, bar, st + 2 * p.a_bytes, 0, k0, n0 / 64);
                    if (p.b_lo)
                        h_tma_3d<kPair>(&map_bl, bar, st + 2 * p.a_bytes + p.b_bytes, 0, k0,
                                        n0 / 64);
                }
            }
        }
        if (p.pace) h_pace_done(p.prog);
    } else if (warp == kHWarpMma && leader) {
        // descriptors of stage 0, K-step 0; per-stage / per-K-step / plane
        // offsets in 16-byte units (start-address field never carries: < 228 KB)
        const uint64_t a0 = p.a_kmajor ? make_desc(smem0, 16u, 1024u, kLayoutSW128)
                                       : make_desc(smem0, kHChunkBytes, 1024u, kLayoutSW128);
        const uint64_t b0 = p.b_kmajor ? make_desc(smem0 + 2 * p.a_bytes, 16u, 1024u, kLayoutSW128)
                                       : make_desc(smem0 + 2 * p.a_bytes, kHChunkBytes, 1024u,
                                                   kLayoutSW128);
        const uint64_t sstep = p.stage_bytes >> 4;
        const uint64_t ajstep = p.a_kmajor ? (32u >> 4) : (2048u >> 4);  // 16 K: +32 B | +2 rows groups
        const uint64_t bjstep = p.b_kmajor ? (32u >> 4) : (2048u >> 4);
        const uint64_t alo = p.a_bytes >> 4, blo = p.b_bytes >> 4;
        // Accumulation chunks of chunk_kb K blocks alternate between the two
        // TMEM buffers; the epilogue adds each finished chunk into registers
        // (fp32, round to nearest) while the next one accumulates.  The
        // tensor core's own fp32 accumulation truncates, so its error grows
        // with the chain length (K = 262144 in one chain: -3e-5 relative on
        // positive data, about -1e-4 on sigma at C3); chains of 1024 keep it
        // at ~7e-6 there (measured: 512 -> 3.3e-6, 64 -> 2.3e-7).
        Ring r;
        int cc = 0;
        for (int u = ustart; u < units; u += ustride) {
            const HWork w = h_unit<kPair>(p, u);
            for (int c0 = w.kb0; c0 < w.kb1; c0 += p.chunk_kb, ++cc) {
                const int buf = cc & 1;
                const uint32_t aph = (uint32_t)(cc >> 1) & 1u;
                mbar_wait(&tempty[buf], aph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + (uint32_t)(buf * p.acc_stride);
                const int c1 = min(c0 + p.chunk_kb, w.kb1);
                for (int kb = c0; kb < c1; ++kb, r.next(S)) {
                    const int s = r.s;
                    mbar_wait(&full[s], r.ph);
                    tc_fence_after();
                    const uint64_t as = a0 + (uint64_t)s * sstep, bs = b0 + (uint64_t)s * sstep;
#pragma unroll
                    for (int j = 0; j < kHKSteps; ++j) {
                        const uint32_t acc = (kb > c0 || j > 0) ? 1u : 0u;
                        const uint64_t ah = as + (uint64_t)j * ajstep, bh = bs + (uint64_t)j * bjstep;
                        h_mma<kPair>(d, ah + alo, bh, p.idesc, acc);  // a_lo b_hi
                        if (p.b_lo) h_mma<kPair>(d, ah, bh + blo, p.idesc, 1u);  // a_hi b_lo
                        h_mma<kPair>(d, ah, bh, p.idesc, 1u);         // a_hi b_hi
                    }
                    if (kPair) tc_commit_pair_e(&empty[s]);
                    else tc_commit_e(&empty[s]);
                }
                if (kPair) tc_commit_pair_e(&tfull[buf]);
                else tc_commit_e(&tfull[buf]);
            }
        }
    } else if (warp >= kHWarpEpi) {
        // 12 warps: TMEM lane quadrant q = warp % 4, column part = which 4 of them
        const int q = warp & 3;
        const int part = (warp - kHWarpEpi) >> 2;
        const int ng = p.bn / 16, per = (ng + kHEpiParts - 1) / kHEpiParts;
        const int g0 = part * per;                               // first 16-column group
        const int g1 = min(ng, g0 + per);                        // past the last
        // 2^-(ea+eb), applied as two exact power-of-two factors
        const int ea = __ldg(p.a_e), eb = __ldg(p.b_e);
        const float sc = ldexpf(1.f, -ea) * ldexpf(1.f, -eb);
        const float alpha = p.alpha * sc;
        float emit_scale = 0.f;
        bool emit_bad = false;
        if (p.emit_hi) {
            const int e_out = p.emit_fixed ? p.emit_e_fixed : ea + eb - p.emit_shift;
            emit_scale = p.alpha * ldexpf(ldexpf(1.f, e_out - ea), -eb);
            if (blockIdx.x == 0 && warp == kHWarpEpi && lane == 0) *p.emit_e = e_out;
        }
        int cc = 0;
        for (int u = ustart; u < units; u += ustride) {
            const HWork w = h_unit<kPair>(p, u);
            float acc[kEC][16];
#pragma unroll
            for (int i = 0; i < kEC; ++i)
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[i][e] = 0.f;
            for (int c0 = w.kb0; c0 < w.kb1; c0 += p.chunk_kb, ++cc) {
                const int buf = cc & 1;
                const uint32_t aph = (uint32_t)(cc >> 1) & 1u;
                mbar_wait_idle(&tfull[buf], aph);
                tc_fence_after();
                const uint32_t tbase =
                    tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * p.acc_stride);
#pragma unroll
                for (int i = 0; i < kEC; ++i) {
                    if (g0 + i < g1) {
                        float v[16];
                        tmem_ld16(tbase + 16u * (uint32_t)(g0 + i), v);
                        acc_add16(acc[i], v);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (kPair) mbar_arrive_cluster_e(tempty_cl0 + 8u * (uint32_t)buf);
                else mbar_arrive_e(&tempty[buf]);
            }
            const int row = w.tm * kRowsPerUnit + (int)rank * HM + q * 32 + lane;
            if (row >= p.M) continue;
            if (p.emit_hi) {
                // C^T split: for each column, the warp's 32 rows are 64
                // contiguous bytes of each plane
#pragma unroll
                for (int i = 0; i < kEC; ++i) {
                    const int col0 = w.tn * p.bn + 16 * (g0 + i);
                    if (g0 + i >= g1 || col0 >= p.N) continue;
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        if (col0 + e < p.N) {
                            const float v = emit_scale * acc[i][e];
                            emit_bad |= !(fabsf(v) < 65504.f);  // (NaN included)
                            const __half h = __float2half_rn(v);
                            const size_t o = (size_t)(col0 + e) * p.emit_ld + row;
                            p.emit_hi[o] = h;
                            p.emit_lo[o] = __float2half_rn(v - __half2float(h));
                        }
                    }
                }
                continue;
            }
#pragma unroll
            for (int i = 0; i < kEC; ++i) {
                const int col0 = w.tn * p.bn + 16 * (g0 + i);
                if (g0 + i >= g1 || col0 >= p.N) continue;
                const int lim = min(16, p.N - col0);
                if (p.splits > 1) {
                    float* dst = p.ws + ((size_t)w.ks * p.M + row) * p.N + col0;
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (e < lim) dst[e] = sc * acc[i][e];
                } else {
                    float* dst = p.C + (size_t)row * p.ldc + col0;
                    const bool vec = lim == 16 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
                    if (vec) {
#pragma unroll
                        for (int e = 0; e < 16; e += 4) {
                            float4 o = make_float4(alpha * acc[i][e], alpha * acc[i][e + 1],
                                                   alpha * acc[i][e + 2], alpha * acc[i][e + 3]);
                            if (p.beta != 0.f) {
                                const float4 c = *reinterpret_cast<float4*>(dst + e);
                                o.x += p.beta * c.x; o.y += p.beta * c.y;
                                o.z += p.beta * c.z; o.w += p.beta * c.w;
                            }
                            *reinterpret_cast<float4*>(dst + e) = o;
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            if (e < lim)
                                dst[e] = p.beta != 0.f ? alpha * acc[i][e] + p.beta * dst[e]
                                                       : alpha * acc[i][e];
                    }
                }
            }
        }
        if (p.emit_hi && p.overflow && emit_bad) atomicOr(p.overflow, 1);
    }
    tc_fence_before();
    if (kPair) cluster_sync_all();
    else __syncthreads();
    if (warp == kHWarpMma) {
        tc_fence_after();
        if (kPair)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(kHTmemCols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(kHTmemCols));
    }
}

__global__ void h3_splitk_reduce(const float* __restrict__ ws, int splits, int64_t M, int64_t N,
                                 float alpha, float beta, float* __restrict__ C, int64_t ldc) {
    const int64_t total = M * N;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int z = 0; z < splits; ++z) s += ws[(int64_t)z * total + t];
        const int64_t i = t / N, j = t - i * N;
        float* c = C + i * ldc + j;
        *c = beta == 0.f ? alpha * s : alpha * s + beta * *c;
    }
}

// ------------------------------------------------------------- the split --
// e = 15 - E for max|X| = f 2^E (f in [0.5, 1)): max|X| 2^e in [2^14, 2^15).
// All-zero or non-finite max: e = 0 (non-finite inputs are rejected upstream).
__device__ __forceinline__ int h2_exponent(uint32_t amax_bits) {
    const float a = __uint_as_float(amax_bits);
    if (!(a > 0.f) || !isfinite(a)) return 0;
    int E;
    frexpf(a, &E);
    return min(15 - E, 126);
}
__device__ __forceinline__ void h2_pair(float x, float s, __half& hi, __half& lo) {
    const float xs = x * s;  // exact: a power of two
    hi = __float2half_rn(xs);
    lo = __float2half_rn(xs - __half2float(hi));  // the difference is exact in fp32
}

__global__ void absmax_kernel(const float* __restrict__ X, int64_t rows, int64_t cols, int64_t ld,
                              uint32_t* __restrict__ amax) {
    uint32_t m = 0;
    const int64_t c4 = (cols + 3) / 4;
    const bool vec = (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows * c4;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / c4, j = (t - i * c4) * 4;
        const float* x = X + i * ld + j;
        if (vec && j + 4 <= cols) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(x));
            m = max(m, max(max(__float_as_uint(fabsf(v.x)), __float_as_uint(fabsf(v.y))),
                           max(__float_as_uint(fabsf(v.z)), __float_as_uint(fabsf(v.w)))));
        } else {
            for (int64_t k = j; k < cols && k < j + 4; ++k)
                m = max(m, __float_as_uint(fabsf(x[k - j])));
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(amax, m);
}

// out (rows x cols, ldh) = split of X, 4 elements per thread
__global__ void split_h2_kernel(const float* __restrict__ X, int64_t rows, int64_t cols, int64_t ld,
                                const uint32_t* __restrict__ amax, __half* __restrict__ hi,
                                __half* __restrict__ lo, int64_t ldh, int* __restrict__ e_out) {
    const int e = h2_exponent(*amax);
    const float s = ldexpf(1.f, e);
    if (blockIdx.x == 0 && threadIdx.x == 0) *e_out = e;
    const int64_t c4 = (cols + 3) / 4;
    const bool vec = (ld & 3) == 0 && (ldh & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(hi) & 7) == 0 &&
                     (reinterpret_cast<uintptr_t>(lo) & 7) == 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows * c4;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / c4, j = (t - i * c4) * 4;
        const float* x = X + i * ld + j;
        if (vec && j + 4 <= cols) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(x));
            __half h[4], l[4];
            h2_pair(v.x, s, h[0], l[0]);
            h2_pair(v.y, s, h[1], l[1]);
            h2_pair(v.z, s, h[2], l[2]);
            h2_pair(v.w, s, h[3], l[3]);
            *reinterpret_cast<uint2*>(hi + i * ldh + j) = *reinterpret_cast<uint2*>(h);
            *reinterpret_cast<uint2*>(lo + i * ldh + j) = *reinterpret_cast<uint2*>(l);
        } else {
            for (int64_t k = j; k < cols && k < j + 4; ++k)
                h2_pair(x[k - j], s, hi[i * ldh + k], lo[i * ldh + k]);
        }
    }
}

// In place: row i of X (ld fp32 = 4 ld bytes) becomes [hi (cols halves) ... |
// lo at half offset ld ...]: the planes' leading dimension is 2 ld halves.
// One CTA per row at a time: the row is staged in shared memory first.
__global__ void __launch_bounds__(256)
split_h2_inplace_kernel(float* __restrict__ X, int64_t rows, int64_t cols, int64_t ld,
                        const uint32_t* __restrict__ amax, int* __restrict__ e_out) {
    extern __shared__ __align__(16) float srow[];
    const int e = h2_exponent(*amax);
    const float s = ldexpf(1.f, e);
    if (blockIdx.x == 0 && threadIdx.x == 0) *e_out = e;
    const int64_t c4 = cols / 4;
    for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
        float* x = X + i * ld;
        for (int64_t j = threadIdx.x; j < c4; j += blockDim.x)
            reinterpret_cast<float4*>(srow)[j] = reinterpret_cast<const float4*>(x)[j];
        for (int64_t j = c4 * 4 + threadIdx.x; j < cols; j += blockDim.x) srow[j] = x[j];
        __syncthreads();
        __half* hi = reinterpret_cast<__half*>(x);
        __half* lo = hi + ld;
        for (int64_t j = threadIdx.x; j < (cols + 3) / 4; j += blockDim.x) {
            const int64_t k = 4 * j;
            __half h[4], l[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (k + u < cols) h2_pair(srow[k + u], s, h[u], l[u]);
                else h[u] = l[u] = __float2half_rn(0.f);
            }
            reinterpret_cast<uint2*>(hi)[j] = *reinterpret_cast<uint2*>(h);  // 8-byte stores
            reinterpret_cast<uint2*>(lo)[j] = *reinterpret_cast<uint2*>(l);
        }
        __syncthreads();
    }
}

// out (cols x rows, ldh) = split of X^T: 64 x 64 tiles through shared memory
__global__ void __launch_bounds__(256)
split_h2_t_kernel(const float* __restrict__ X, int64_t rows, int64_t cols, int64_t ld,
                  const uint32_t* __restrict__ amax, __half* __restrict__ hi,
                  __half* __restrict__ lo, int64_t ldh, int* __restrict__ e_out) {
    __shared__ float tile[64][65];
    const int e = h2_exponent(*amax);
    const float s = ldexpf(1.f, e);
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *e_out = e;
    const int64_t r0 = (int64_t)blockIdx.y * 64, c0 = (int64_t)blockIdx.x * 64;
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
    for (int k = ty; k < 64; k += 4) {
        const int64_t i = r0 + k, j = c0 + tx;
        tile[k][tx] = (i < rows && j < cols) ? __ldg(X + i * ld + j) : 0.f;
    }
    __syncthreads();
    // output row c0 + k holds X[r0 .. r0+63, c0 + k]; a thread writes 2 elements
    const int tx2 = threadIdx.x & 31, ty2 = threadIdx.x >> 5;  // 32 x 8
    for (int k = ty2; k < 64; k += 8) {
        const int64_t orow = c0 + k, oc = r0 + 2 * tx2;
        if (orow >= cols || oc >= rows) continue;
        __half h0, l0, h1, l1;
        h2_pair(tile[2 * tx2][k], s, h0, l0);
        h2_pair(tile[2 * tx2 + 1][k], s, h1, l1);
        if (oc + 1 < rows && (ldh & 1) == 0) {
            *reinterpret_cast<__half2*>(hi + orow * ldh + oc) = __halves2half2(h0, h1);
            *reinterpret_cast<__half2*>(lo + orow * ldh + oc) = __halves2half2(l0, l1);
        } else {
            hi[orow * ldh + oc] = h0;
            lo[orow * ldh + oc] = l0;
            if (oc + 1 < rows) {
                hi[orow * ldh + oc + 1] = h1;
                lo[orow * ldh + oc + 1] = l1;
            }
        }
    }
}


// ---------------------------------------------- 3xFP16 with an in-kernel A split --
// gemm_h3s: the same products with A given in FP32 -- for the one big
// product whose left operand is read once (randsvd's B^T = A^T Q, A = the
// m x n input itself, too large to pre-split: a split pass would cost more
// HBM time than it saves).  op(A) = A^T with A stored K x M (MN-major),
// exponent 2^ea from the caller (a bound on max|A|); B pre-split (K-major
// planes).  Warps: 0 TMA (fp32 A tile as [4 chunks][HK k][32 m], B hi/lo
// planes), 1 MMA (kind::f16 with A from TENSOR MEMORY), 2-5 split (thread =
// tile row: 64 fp32 -> (hi, lo) fp16 pairs -> tcgen05.st into the stage's TMEM
// slot), 6-9 epilogue.  TMEM: [accumulator | A slots of 64 columns: 32 hi |
// 32 lo].  A value that does not fit fp16 after scaling sets *overflow (the
// caller then recomputes with 3xTF32).
// 8 split warps: two per TMEM lane quadrant, each converting half of the
// stage's 64 K rows (with 4, the split of stage s+1 did not finish within
// stage s's MMAs: tensor pipe 77% active at C5)
constexpr int kSWarpTma = 0, kSWarpMma = 1, kSWarpAx = 2, kSNumXf = 8,
              kSWarpEpi = kSWarpAx + kSNumXf, kSNumEpi = 8;
constexpr int kSThreads = 32 * (kSWarpEpi + kSNumEpi);
constexpr int kSEpiCols = 6;                     // 16-column groups per epilogue thread
constexpr int kSMaxBn = 2 * 16 * kSEpiCols;      // 192
constexpr int kSSlots = 2;                       // TMEM A slots (the smem ring runs deeper)
constexpr uint32_t kSSlotCols = 64;              // 32 hi | 32 lo (2 fp16 per column)
constexpr uint32_t kSChunkBytes = 32 * HK * 4;   // fp32 A: 32 M x HK K per box chunk

struct H3SParams {
    int M, N, K;
    int bn, tiles_m, tiles_n, splits, kb_per_split, num_kb;
    float alpha, beta;
    float* C;
    long long ldc;
    float* ws;
    int stages;
    uint32_t a_bytes, b_bytes, stage_bytes;
    uint32_t idesc;
    int acc_stride;
    const int* a_e;
    const int* b_e;
    int* overflow;
    int chunk_kb;
    unsigned* prog;  // pacing slots (see h_pace), or null
    int pace;
};

__device__ __forceinline__ HWork hs_unit(const H3SParams& p, int u) {
    HWork w;
    w.tn = u % p.tiles_n;
    const int r = u / p.tiles_n;
    w.tm = r % p.tiles_m;
    w.ks = r / p.tiles_m;
    w.kb0 = w.ks * p.kb_per_split;
    w.kb1 = min(w.kb0 + p.kb_per_split, p.num_kb);
    return w;
}

// D[tmem] (+)= A[tmem] * B[smem desc], kind::f16
template <bool kPair>
__device__ __forceinline__ void hs_mma(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
    if (kPair)
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t.reg .b32 r;\n\t"
            "setp.ne.b32 q, %4, 0;\n\t"
            "elect.sync r|p, 0xffffffff;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, q;\n\t}" ::"r"(d),
            "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t.reg .b32 r;\n\t"
            "setp.ne.b32 q, %4, 0;\n\t"
            "elect.sync r|p, 0xffffffff;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, q;\n\t}" ::"r"(d),
            "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
}

// two fp32 values (already scaled) -> packed fp16 hi pair and lo pair
__device__ __forceinline__ void h2_split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(x0, x1);     // .x (low half) = x0
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}

template <bool kPair>
__global__ void __launch_bounds__(kSThreads, 1)
gemm_h3s_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_bh,
                const __grid_constant__ CUtensorMap map_bl, const H3SParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * p.stage_bytes);
    uint64_t* full = bars;                 // [S] smem stage landed (TMA)
    uint64_t* empty = bars + S;            // [S] smem stage consumed (MMA commit)
    uint64_t* split = bars + 2 * S;        // [2] TMEM A slot written (split warps)
    uint64_t* slotfree = split + kSSlots;  // [2] TMEM A slot consumed (MMA commit)
    uint64_t* tfull = slotfree + kSSlots;  // [2] accumulator chunk done (MMA commit)
    uint64_t* tempty = tfull + 2;          // [2] accumulator drained (epilogue)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int units = p.tiles_m * p.tiles_n * p.splits;
    const uint32_t rank = kPair ? cluster_rank() : 0u;
    const bool leader = rank == 0;
    const int ustart = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int ustride = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    constexpr int kRowsPerUnit = kPair ? 2 * HM : HM;
    constexpr int kNumXf = kSNumXf;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int t = 0; t < kSSlots; ++t) {
            // paired: the peer's MMA warp forwards its split warps' completion
            // as ONE cluster arrive on the leader's split[t]
            mbar_init(&split[t], (kPair && leader) ? kNumXf + 1 : kNumXf);
            mbar_init(&slotfree[t], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kPair ? 2 * kSNumEpi : kSNumEpi);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kSWarpMma) {
        if (kPair) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kHTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kHTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    if (kPair) cluster_sync_all();
    else __syncthreads();
    tc_fence_after();
    const uint32_t split_cl0 = kPair ? mapa_shared(smem_u32(split), 0) : 0u;
    const uint32_t tempty_cl0 = kPair ? mapa_shared(smem_u32(tempty), 0) : 0u;
    const uint32_t tmem_base = *tmem_slot;
    // TMEM: [accumulator 0 | accumulator 1 | A slot 0 | A slot 1]
    const uint32_t acol0 = 2u * (uint32_t)p.acc_stride;
    const uint32_t smem0 = smem_u32(smem);

    if (warp == kSWarpTma) {
        Ring r;
        const int bcols = kPair ? p.bn / 2 : p.bn;
        unsigned wave = 0;
        int lo_cache = 0;
        for (int u = ustart; u < units; u += ustride, ++wave) {
            const HWork w = hs_unit(p, u);
            const int m0 = w.tm * kRowsPerUnit + (int)rank * HM;
            const int n0 = w.tn * p.bn + (int)rank * bcols;
            for (int kb = w.kb0; kb < w.kb1; ++kb, r.next(S)) {
                const int s = r.s;
                if (p.pace && ((kb - w.kb0) & 3) == 0)
                    h_pace(p.prog, p.pace, wave, kb - w.kb0, lo_cache);
                mbar_wait(&empty[s], r.ph ^ 1);
                mbar_expect_tx_e(&full[s], p.stage_bytes);
                const uint32_t st = smem0 + (uint32_t)s * p.stage_bytes;
                const uint32_t bar = smem_u32(&full[s]);
                const int k0 = kb * HK;
                h_tma_3d<false>(&map_a, bar, st, 0, k0, m0 / 32);
                h_tma_2d<false>(&map_bh, bar, st + p.a_bytes, k0, n0);
                h_tma_2d<false>(&map_bl, bar, st + p.a_bytes + p.b_bytes, k0, n0);
            }
        }
        if (p.pace) h_pace_done(p.prog);
    } else if (warp == kSWarpMma && leader) {
        // accumulation chunks alternate between the two TMEM accumulators and
        // are summed in registers by the epilogue (see gemm_h3_kernel)
        const uint64_t b0 = make_desc(smem0 + p.a_bytes, 16u, 1024u, kLayoutSW128);
        const uint64_t sstep = p.stage_bytes >> 4;
        const uint64_t bjstep = 32u >> 4;
        const uint64_t blo = p.b_bytes >> 4;
        Ring r, rt;
        int cc = 0;
        for (int u = ustart; u < units; u += ustride) {
            const HWork w = hs_unit(p, u);
            for (int c0 = w.kb0; c0 < w.kb1; c0 += p.chunk_kb, ++cc) {
                const int buf = cc & 1;
                mbar_wait(&tempty[buf], ((uint32_t)(cc >> 1) & 1u) ^ 1u);
                tc_fence_after();
                const uint32_t d = tmem_base + (uint32_t)(buf * p.acc_stride);
                const int c1 = min(c0 + p.chunk_kb, w.kb1);
                for (int kb = c0; kb < c1; ++kb, r.next(S), rt.next(kSSlots)) {
                    const int s = r.s, t = rt.s;
                    mbar_wait(&split[t], rt.ph);  // implies stage s landed
                    tc_fence_after();
                    const uint64_t bs = b0 + (uint64_t)s * sstep;
                    const uint32_t ah = tmem_base + acol0 + kSSlotCols * (uint32_t)t;
#pragma unroll
                    for (int j = 0; j < kHKSteps; ++j) {
                        const uint32_t acc = (kb > c0 || j > 0) ? 1u : 0u;
                        const uint32_t a_hi = ah + 8u * j, a_lo = a_hi + 32u;
                        const uint64_t bh = bs + (uint64_t)j * bjstep;
                        hs_mma<kPair>(d, a_lo, bh, p.idesc, acc);      // a_lo b_hi
                        hs_mma<kPair>(d, a_hi, bh + blo, p.idesc, 1u); // a_hi b_lo
                        hs_mma<kPair>(d, a_hi, bh, p.idesc, 1u);       // a_hi b_hi
                    }
                    if (kPair) {
                        tc_commit_pair_e(&empty[s]);
                        tc_commit_pair_e(&slotfree[t]);
                    } else {
                        tc_commit_e(&empty[s]);
                        tc_commit_e(&slotfree[t]);
                    }
                }
                if (kPair) tc_commit_pair_e(&tfull[buf]);
                else tc_commit_e(&tfull[buf]);
            }
        }
    } else if (kPair && warp == kSWarpMma) {
        // peer CTA: forward "slot t split done" to the leader's split[t]
        Ring rt;
        for (int u = ustart; u < units; u += ustride) {
            const HWork w = hs_unit(p, u);
            for (int kb = w.kb0; kb < w.kb1; ++kb, rt.next(kSSlots)) {
                mbar_wait(&split[rt.s], rt.ph);
                mbar_arrive_cluster_e(split_cl0 + 8u * (uint32_t)rt.s);
            }
        }
    } else if (warp >= kSWarpAx && warp < kSWarpEpi) {
        // split: thread = tile row (TMEM lane); lane quadrant = warp % 4 = box
        // chunk; the two warps of a quadrant take K rows 0..31 and 32..63
        const int q = warp & 3;
        const int half = (warp - kSWarpAx) >> 2;
        const uint32_t tlane = (uint32_t)(q * 32) << 16;
        const float sa = ldexpf(1.f, __ldg(p.a_e));
        float amax = 0.f;
        Ring r, rt;
        for (int u = ustart; u < units; u += ustride) {
            const HWork w = hs_unit(p, u);
            // rows past M read the row padding (any bits): kept out of the
            // overflow test; their outputs are never stored
            const bool live = w.tm * kRowsPerUnit + (int)rank * HM + q * 32 + lane < p.M;
            for (int kb = w.kb0; kb < w.kb1; ++kb, r.next(S), rt.next(kSSlots)) {
                const int s = r.s, t = rt.s;
                mbar_wait(&full[s], r.ph);
                mbar_wait(&slotfree[t], rt.ph ^ 1);
                tc_fence_after();
                // [chunk q][k][32 m]: lanes read 128 contiguous bytes per k
                const uint32_t cb = smem0 + (uint32_t)s * p.stage_bytes +
                                    (uint32_t)q * kSChunkBytes + (uint32_t)lane * 4u;
                const uint32_t ta = tmem_base + tlane + acol0 + kSSlotCols * (uint32_t)t;
                {
                    uint32_t hi[16], lo[16];
#pragma unroll
                    for (int k2 = 0; k2 < 16; ++k2) {
                        const int k = half * 32 + 2 * k2;
                        const float x0 = __uint_as_float(lds32(cb + 128u * k)) * sa;
                        const float x1 = __uint_as_float(lds32(cb + 128u * (k + 1))) * sa;
                        if (live) amax = fmaxf(amax, fmaxf(fabsf(x0), fabsf(x1)));
                        h2_split2(x0, x1, hi[k2], lo[k2]);
                    }
                    tmem_st16(ta + 16u * half, hi);
                    tmem_st16(ta + 32u + 16u * half, lo);
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                mbar_arrive_e(&split[t]);
            }
        }
        // fp16 holds |x| < 65520 (round to nearest); NaN entries propagate to C
        if (!(amax < 65504.f) && p.overflow) atomicOr(p.overflow, 1);
    } else if (warp >= kSWarpEpi) {
        // 8 warps: TMEM lane quadrant q = warp % 4, column half = which 4 of them
        const int q = warp & 3;
        const int part = (warp - kSWarpEpi) >> 2;
        const int ng = p.bn / 16, per = (ng + 1) / 2;
        const int g0 = part * per, g1 = min(ng, g0 + per);
        const float sc = ldexpf(1.f, -__ldg(p.a_e)) * ldexpf(1.f, -__ldg(p.b_e));
        const float alpha = p.alpha * sc;
        int cc = 0;
        for (int u = ustart; u < units; u += ustride) {
            const HWork w = hs_unit(p, u);
            float acc[kSEpiCols][16];
#pragma unroll
            for (int i = 0; i < kSEpiCols; ++i)
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[i][e] = 0.f;
            for (int c0 = w.kb0; c0 < w.kb1; c0 += p.chunk_kb, ++cc) {
                const int buf = cc & 1;
                mbar_wait_idle(&tfull[buf], (uint32_t)(cc >> 1) & 1u);
                tc_fence_after();
                const uint32_t tbase =
                    tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * p.acc_stride);
#pragma unroll
                for (int i = 0; i < kSEpiCols; ++i) {
                    if (g0 + i < g1) {
                        float v[16];
                        tmem_ld16(tbase + 16u * (uint32_t)(g0 + i), v);
                        acc_add16(acc[i], v);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (kPair) mbar_arrive_cluster_e(tempty_cl0 + 8u * (uint32_t)buf);
                else mbar_arrive_e(&tempty[buf]);
            }
            const int row = w.tm * kRowsPerUnit + (int)rank * HM + q * 32 + lane;
            if (row >= p.M) continue;
#pragma unroll
            for (int i = 0; i < kSEpiCols; ++i) {
                const int col0 = w.tn * p.bn + 16 * (g0 + i);
                if (g0 + i >= g1 || col0 >= p.N) continue;
                const int lim = min(16, p.N - col0);
                if (p.splits > 1) {
                    float* dst = p.ws + ((size_t)w.ks * p.M + row) * p.N + col0;
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (e < lim) dst[e] = sc * acc[i][e];
                } else {
                    float* dst = p.C + (size_t)row * p.ldc + col0;
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (e < lim)
                            dst[e] = p.beta != 0.f ? alpha * acc[i][e] + p.beta * dst[e]
                                                   : alpha * acc[i][e];
                }
            }
        }
    }
    tc_fence_before();
    if (kPair) cluster_sync_all();
    else __syncthreads();
    if (warp == kSWarpMma) {
        tc_fence_after();
        if (kPair)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(kHTmemCols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(kHTmemCols));
    }
}

// e_io[0] = 15 - E - margin for max|X| = f 2^E (max from e_io[1]'s bits)
__global__ void h2_exponent_kernel(int* e_io, int margin) {
    if (threadIdx.x == 0) {
        const float a = __uint_as_float((uint32_t)e_io[1]);
        int e = 0;
        if (a > 0.f && isfinite(a)) {
            int E;
            frexpf(a, &E);
            e = min(15 - E - margin, 126);
        }
        e_io[0] = e;
    }
}

// ----------------------------------------------------------------- host ----
PFN_cuTensorMapEncodeTiled_v12000 h_encode = nullptr;
int h_state = -1;
int h_sms = 148;

bool h_init() {
    if (h_state >= 0) return h_state == 1;
    h_state = 0;
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cudaDeviceGetAttribute(&h_sms, cudaDevAttrMultiProcessorCount, dev);
    if (major != 10 || minor != 0) return false;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
        return false;
    h_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    h_state = 1;
    return true;
}

// K-major fp16 [rows x cols] (cols = K contiguous), box {64, box_rows}, SWIZZLE_128B
bool h_encode_k(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t ld,
                uint32_t box_rows) {
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {(cuuint32_t)HK, box_rows};
    cuuint32_t es[2] = {1, 1};
    return h_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// MN-major fp16 A stored [K x M] (M contiguous) as {64, K, M/64 chunks}: one
// box {64, HK, 2} = the CTA's 128 M x HK K tile as [chunk][k][64], SWIZZLE_128B
bool h_encode_mn(CUtensorMap* map, const void* base, uint64_t m, uint64_t k, uint64_t ld,
                 uint32_t box_mn = HM) {
    cuuint64_t dims[3] = {64, k, (cuuint64_t)cdiv((int64_t)m, 64)};
    cuuint64_t strides[2] = {ld * 2, 128};
    cuuint32_t box[3] = {64, (cuuint32_t)HK, box_mn / 64};
    cuuint32_t es[3] = {1, 1, 1};
    return h_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct HPlan {
    int bn, tiles_m, tiles_n, splits, num_kb, kb_per_split, stages, acc_stride;
    uint32_t a_bytes, b_bytes, stage_bytes;
    size_t smem;
};

// K blocks per accumulation chunk (chains of 1024): see the MMA role
int h_chunk_kb() {
    return 16;
}

bool h_pair(int64_t M) {
    return M > HM;
}

HPlan h_plan(int64_t M, int64_t N, int64_t K, int64_t ws_cap_elems, bool pair, bool b_lo = true) {
    HPlan pl;
    const int max_bn = pair ? kHMaxBn : 128;
    pl.tiles_n = (int)cdiv(N, max_bn);
    pl.bn = (int)(cdiv(cdiv(N, pl.tiles_n), 16) * 16);
    pl.tiles_m = (int)cdiv(M, pair ? 2 * HM : HM);
    pl.num_kb = (int)cdiv(K, HK);
    const int slots_machine = pair ? h_sms / 2 : h_sms;
    const int64_t base = (int64_t)pl.tiles_m * pl.tiles_n;
    int splits = 1;
    if (base < 4 * slots_machine) {
        double best = 0;
        const int maxs = (int)std::max<int64_t>(1, pl.num_kb / 4);
        for (int s = 1; s <= std::min(64, maxs); ++s) {
            const int64_t units = base * s;
            if (s > 1 && (int64_t)s * M * N > ws_cap_elems) break;
            const double waves = (double)cdiv(units, slots_machine);
            const double eff = (double)units / (waves * slots_machine);
            const double score = std::min(1.0, (double)units / slots_machine) * eff;
            if (score > best + 0.02) { best = score; splits = s; }
        }
    }
    pl.kb_per_split = (int)cdiv(pl.num_kb, splits);
    pl.splits = (int)cdiv(pl.num_kb, pl.kb_per_split);
    pl.a_bytes = HM * HK * 2;
    const int bcols = pair ? pl.bn / 2 : pl.bn;
    pl.b_bytes = (uint32_t)bcols * HK * 2;
    pl.stage_bytes = 2 * pl.a_bytes + (b_lo ? 2 : 1) * pl.b_bytes;
    pl.acc_stride = (int)cdiv(pl.bn, 32) * 32;
    const size_t budget = 227 * 1024;
    const int st = (int)((budget - 1024 - 256) / pl.stage_bytes);
    pl.stages = std::max(2, std::min(kHMaxStages, st));
    pl.smem = 1024 + (size_t)pl.stages * pl.stage_bytes + (2 * pl.stages + 4) * 8 + 16;
    return pl;
}


// fp32 A stored [K x M] (M contiguous) as {32, K, M/32 chunks}: one box
// {32, HK, 4} = the CTA's 128 M x HK K tile as [chunk][k][32], unswizzled (the
// split warps read it row-per-lane)
bool hs_encode_a(CUtensorMap* map, const float* base, uint64_t m, uint64_t k, uint64_t ld) {
    cuuint64_t dims[3] = {32, k, (cuuint64_t)cdiv((int64_t)m, 32)};
    cuuint64_t strides[2] = {ld * 4, 128};
    cuuint32_t box[3] = {32, (cuuint32_t)HK, (cuuint32_t)(HM / 32)};
    cuuint32_t es[3] = {1, 1, 1};
    return h_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims,
                    strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

HPlan hs_plan(int64_t M, int64_t N, int64_t K, int64_t ws_cap_elems, bool pair) {
    HPlan pl = h_plan(M, N, K, ws_cap_elems, pair);
    pl.a_bytes = HM * HK * 4;
    pl.stage_bytes = pl.a_bytes + 2 * pl.b_bytes;
    const size_t budget = 227 * 1024;
    const int st = (int)((budget - 1024 - 512) / pl.stage_bytes);
    pl.stages = std::max(2, std::min(kHMaxStages, st));
    pl.smem = 1024 + (size_t)pl.stages * pl.stage_bytes + (2 * pl.stages + 2 * kSSlots + 4) * 8 + 16;
    return pl;
}
}  // namespace

constexpr int64_t kPaceBytes = 1024;  // pacing slots (<= 256 CTAs) at the head of ws
constexpr int kPaceKb = 32;            // K blocks a producer may lead its wave by (SYRK;
constexpr int kPaceKbS = 64;           // K4s, whose wave reads ~1 MB per K block, 64)
constexpr int kPaceMinKb = 512;        // units shorter than this are not paced
constexpr int kPaceKbProd = 16;        // the products' units (K = l ~ 125 K blocks)
constexpr int kPaceMinKbProd = 64;

int64_t gemm_h3_ws_bytes(int ta, int64_t M, int64_t N, int64_t K) {
    (void)ta;
    if (!h_init()) return 0;
    const HPlan pl = h_plan(M, N, K, INT64_MAX, h_pair(M));
    return kPaceBytes + (pl.splits > 1 ? (int64_t)pl.splits * M * N * 4 : 0);
}

struct H3Emit {
    void* hi;
    void* lo;
    int64_t ld;
    int shift, fixed, e_fixed;
    int32_t* e_out;
    int32_t* overflow;
    int b_lower;  // B (stored N x K) is lower triangular: skip the K blocks past each N tile
};

int gemm_h3_impl(int ta, int64_t M, int64_t N, int64_t K, float alpha, const void* Ahi,
                 const void* Alo, int64_t lda, const int32_t* a_e, const void* Bhi, const void* Blo,
                 int64_t ldb, const int32_t* b_e, float beta, float* C, int64_t ldc, void* ws,
                 int64_t ws_bytes, const H3Emit* emit, cudaStream_t st, bool b_lo = true) {
    if (!h_init()) {
        set_error("unsupported: the 3xFP16 tcgen05 GEMM needs an sm_100 device");
        return SKP_ERR_UNSUPPORTED;
    }
    if (M == 0 || N == 0) return SKP_OK;
    if (K == 0 || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) {
        set_error("unsupported: gemm_h3 sizes");
        return SKP_ERR_UNSUPPORTED;
    }
    b_lo = b_lo && Blo != nullptr;  // no lo plane: 2 products, B rounded to fp16
    const uintptr_t al = reinterpret_cast<uintptr_t>(Ahi) | reinterpret_cast<uintptr_t>(Alo) |
                         reinterpret_cast<uintptr_t>(Bhi) | reinterpret_cast<uintptr_t>(Blo);
    if ((al & 15) || (lda & 7) || (ldb & 7) || (ta && (lda & 63))) {
        set_error("unsupported: gemm_h3 needs 16-byte aligned planes, ld %% 8 == 0 (%% 64 for "
                  "MN-major A): lda=%lld ldb=%lld", (long long)lda, (long long)ldb);
        return SKP_ERR_UNSUPPORTED;
    }
    const bool pair = h_pair(M);
    // ws: [pacing slots | split-K partials]
    unsigned* prog = (ws && ws_bytes >= kPaceBytes) ? reinterpret_cast<unsigned*>(ws) : nullptr;
    void* wsp = prog ? reinterpret_cast<char*>(ws) + kPaceBytes : ws;
    const int64_t wsp_bytes = prog ? ws_bytes - kPaceBytes : ws_bytes;
    const int64_t cap = (wsp && !emit) ? wsp_bytes / 4 : 0;  // emit: no split-K partials
    HPlan pl = h_plan(M, N, K, cap, pair, b_lo);
    if (pl.splits > 1 && (!wsp || emit || (int64_t)pl.splits * M * N * 4 > wsp_bytes))
        pl = h_plan(M, N, K, 0, pair, b_lo);
    H3Params p;
    p.b_lo = b_lo ? 1 : 0;
    p.M = (int)M; p.N = (int)N; p.K = (int)K;
    p.bn = pl.bn; p.tiles_m = pl.tiles_m; p.tiles_n = pl.tiles_n; p.splits = pl.splits;
    p.kb_per_split = pl.kb_per_split; p.num_kb = pl.num_kb;
    p.a_kmajor = ta ? 0 : 1;
    p.b_kmajor = 1;
    p.sym = 0;
    p.sym_tiles = 0;
    p.tri_k = 0;
    // pacing: the N tiles of one M block read the same A rows; many waves of
    // units each holding ~100 MB of A in flight (C5's Y = A~ W: 12 M blocks x
    // 8 MB per wave) thrash the L2 (ncu: A~ read 4.7x) unless they move in step
    p.prog = prog;
    p.pace = (prog && pl.kb_per_split >= kPaceMinKbProd) ? kPaceKbProd : 0;
    if (p.pace) SKP_CUDA(cudaMemsetAsync(prog, 0, kPaceBytes, st));
    p.alpha = alpha; p.beta = beta; p.C = C; p.ldc = ldc;
    p.ws = pl.splits > 1 ? reinterpret_cast<float*>(wsp) : nullptr;
    p.stages = pl.stages; p.a_bytes = pl.a_bytes; p.b_bytes = pl.b_bytes;
    p.stage_bytes = pl.stage_bytes; p.acc_stride = pl.acc_stride;
    p.a_e = a_e; p.b_e = b_e;
    p.chunk_kb = h_chunk_kb();
    p.emit_hi = emit ? reinterpret_cast<__half*>(emit->hi) : nullptr;
    p.emit_lo = emit ? reinterpret_cast<__half*>(emit->lo) : nullptr;
    p.emit_ld = emit ? emit->ld : 0;
    p.emit_shift = emit ? emit->shift : 0;
    p.emit_fixed = emit ? emit->fixed : 0;
    p.emit_e_fixed = emit ? emit->e_fixed : 0;
    p.emit_e = emit ? emit->e_out : nullptr;
    p.overflow = emit ? emit->overflow : nullptr;
    p.tri_k = emit ? emit->b_lower : 0;
    // kind::f16 instruction descriptor: D f32, A/B f16, A major from the layout,
    // B K-major, N >> 3, M >> 4
    p.idesc = (1u << 4) | ((uint32_t)(!p.a_kmajor) << 15) | ((uint32_t)(p.bn >> 3) << 17) |
              ((uint32_t)((pair ? 2 * HM : HM) >> 4) << 24);
    CUtensorMap mah, mal, mbh, mbl;
    const int bcols = pair ? p.bn / 2 : p.bn;
    bool ok;
    if (p.a_kmajor)
        ok = h_encode_k(&mah, Ahi, (uint64_t)K, (uint64_t)M, lda, HM) &&
             h_encode_k(&mal, Alo, (uint64_t)K, (uint64_t)M, lda, HM);
    else
        ok = h_encode_mn(&mah, Ahi, (uint64_t)M, (uint64_t)K, lda) &&
             h_encode_mn(&mal, Alo, (uint64_t)M, (uint64_t)K, lda);
    ok = ok && h_encode_k(&mbh, Bhi, (uint64_t)K, (uint64_t)N, ldb, (uint32_t)bcols) &&
         h_encode_k(&mbl, b_lo ? Blo : Bhi, (uint64_t)K, (uint64_t)N, ldb, (uint32_t)bcols);
    if (!ok) {
        set_error("cuTensorMapEncodeTiled failed (gemm_h3)");
        return SKP_ERR_UNSUPPORTED;
    }
    const int units = p.tiles_m * p.tiles_n * p.splits;
    if (pair) {
        SKP_CUDA(cudaFuncSetAttribute(gemm_h3_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(2 * std::min(units, h_sms / 2)));
        cfg.blockDim = dim3(kHThreads);
        cfg.dynamicSmemBytes = pl.smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        SKP_CUDA(cudaLaunchKernelEx(&cfg, gemm_h3_kernel<true>, mah, mal, mbh, mbl, p));
        SKP_LAUNCHED(gemm_h3_kernel_pair);
    } else {
        SKP_CUDA(cudaFuncSetAttribute(gemm_h3_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
        gemm_h3_kernel<false><<<std::min(units, h_sms), kHThreads, pl.smem, st>>>(mah, mal, mbh, mbl,
                                                                                 p);
        SKP_LAUNCHED(gemm_h3_kernel);
    }
    if (p.splits > 1) {
        const int64_t blocks = std::min<int64_t>(cdiv(M * N, 256), (int64_t)h_sms * 8);
        h3_splitk_reduce<<<(unsigned)blocks, 256, 0, st>>>(p.ws, p.splits, M, N, alpha, beta, C,
                                                           ldc);
        SKP_LAUNCHED(h3_splitk_reduce);
    }
    return SKP_OK;
}


// split-K slices for the SYRK: enough units for every CTA pair, and at
// least 64 K blocks (4 promotion chunks) per slice
int syrk_splits(int64_t tiles, int64_t K, int slots) {
    // time ~ waves(tiles s) / s: the smallest, at >= 64 K blocks per slice
    // (C5's Grams: 15 tiles over 74 CTA pairs -> 4 slices in one wave, where
    // 5 slices made 75 units and a second wave for one of them)
    const int64_t nkb = cdiv(K, HK);
    int best = 1;
    double best_t = 1e30;
    for (int s = 1; s <= 16 && (s == 1 || nkb / s >= 64); ++s) {
        const double t = (double)cdiv(tiles * s, (int64_t)slots) / s;
        if (t < best_t - 1e-9) {
            best_t = t;
            best = s;
        }
    }
    return best;
}

struct SyrkPlan {
    HPlan pl;
    int bn, bcols, R, tiles, splits;
    bool pair;
};
SyrkPlan syrk_plan(int64_t N, int64_t K) {
    SyrkPlan sp;
    sp.pair = h_pair(N);
    HPlan& pl = sp.pl;
    pl = h_plan(N, N, K, 0, sp.pair);
    // square tiles: 256 x 256 per CTA pair (each CTA 128 rows of A and 128
    // columns of B; 6 column groups per epilogue thread), 128 x 128 on one CTA
    sp.bn = sp.pair ? 256 : 128;
    sp.bcols = sp.pair ? sp.bn / 2 : sp.bn;
    sp.R = sp.pair ? 2 * HM : HM;
    pl.bn = sp.bn;
    pl.tiles_n = (int)cdiv(N, sp.bn);
    pl.b_bytes = (uint32_t)sp.bcols * HK * 2;
    pl.stage_bytes = 2 * pl.a_bytes + 2 * pl.b_bytes;
    pl.acc_stride = sp.bn;
    pl.stages = std::max(2, std::min(kHMaxStages, (int)((227 * 1024 - 1024 - 256) / pl.stage_bytes)));
    pl.smem = 1024 + (size_t)pl.stages * pl.stage_bytes + (2 * pl.stages + 4) * 8 + 16;
    sp.tiles = 0;
    for (int tm = 0; tm < pl.tiles_m; ++tm)
        sp.tiles += (int)std::min<int64_t>(pl.tiles_n, cdiv((int64_t)(tm + 1) * sp.R, sp.bn));
    sp.splits = syrk_splits(sp.tiles, K, sp.pair ? h_sms / 2 : h_sms);
    pl.kb_per_split = (int)cdiv(pl.num_kb, sp.splits);
    sp.splits = (int)cdiv(pl.num_kb, pl.kb_per_split);
    return sp;
}

int64_t syrk_h3_ws_bytes(int64_t N, int64_t K) {
    if (!h_init() || N == 0 || K == 0) return 0;
    const SyrkPlan sp = syrk_plan(N, K);
    return kPaceBytes + (sp.splits > 1 ? (int64_t)sp.splits * N * N * 4 : 0);
}

// C = alpha A^T A (N x N, symmetric) with A pre-split: stored K x N (N
// contiguous, kmajor = 0: both operands MN-major from the same planes) or
// N x K (kmajor = 1: both K-major, the Gram of the rows of a transposed
// block).  Only the tiles meeting the lower triangle run (~half of the full
// product's MMAs), split over K when there are fewer tiles than CTA pairs;
// the strict upper triangle is then mirrored from the lower one, so C comes
// out exactly symmetric.
__global__ void sym_mirror_kernel(float* __restrict__ C, int64_t N, int64_t ldc) {
    __shared__ float t[32][33];
    const int64_t bi = blockIdx.y, bj = blockIdx.x;  // source tile (bi, bj), bi >= bj
    if (bj > bi) return;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = bi * 32 + r, j = bj * 32 + tx;
        t[r][tx] = (i < N && j < N) ? C[i * ldc + j] : 0.f;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = bj * 32 + r, j = bi * 32 + tx;  // destination (i, j) = source (j, i)
        if (i < N && j < N && j > i) C[i * ldc + j] = t[tx][r];
    }
}

int syrk_h3(int kmajor, int64_t N, int64_t K, float alpha, const void* Ahi, const void* Alo,
            int64_t lda, const int32_t* a_e, float beta, float* C, int64_t ldc, void* ws,
            int64_t ws_bytes, cudaStream_t st) {
    if (!h_init()) {
        set_error("unsupported: the 3xFP16 tcgen05 GEMM needs an sm_100 device");
        return SKP_ERR_UNSUPPORTED;
    }
    if (N == 0) return SKP_OK;
    if (K == 0 || N > INT32_MAX || K > INT32_MAX) {
        set_error("unsupported: syrk_h3 sizes");
        return SKP_ERR_UNSUPPORTED;
    }
    const uintptr_t al = reinterpret_cast<uintptr_t>(Ahi) | reinterpret_cast<uintptr_t>(Alo);
    if ((al & 15) || (kmajor ? (lda & 7) : (lda & 63))) {
        set_error("unsupported: syrk_h3 needs 16-byte aligned planes with lda %% %d == 0 (lda=%lld)",
                  kmajor ? 8 : 64, (long long)lda);
        return SKP_ERR_UNSUPPORTED;
    }
    const SyrkPlan sp = syrk_plan(N, K);
    const HPlan& pl = sp.pl;
    const bool pair = sp.pair;
    const int splits = sp.splits;
    if (!ws || ws_bytes < syrk_h3_ws_bytes(N, K)) {
        set_error("syrk_h3 needs %lld bytes of workspace", (long long)syrk_h3_ws_bytes(N, K));
        return SKP_ERR_ARG;
    }
    unsigned* prog = reinterpret_cast<unsigned*>(ws);
    void* wsp = reinterpret_cast<char*>(ws) + kPaceBytes;
    H3Params p = {};
    p.b_lo = 1;
    p.M = (int)N; p.N = (int)N; p.K = (int)K;
    p.bn = pl.bn; p.tiles_m = pl.tiles_m; p.tiles_n = pl.tiles_n; p.splits = splits;
    p.kb_per_split = pl.kb_per_split; p.num_kb = pl.num_kb;
    p.a_kmajor = kmajor ? 1 : 0;
    p.b_kmajor = kmajor ? 1 : 0;
    p.sym_tiles = sp.tiles;
    p.sym = sp.tiles * splits;
    p.tri_k = 0;
    p.alpha = alpha; p.beta = beta; p.C = C; p.ldc = ldc;
    p.ws = splits > 1 ? reinterpret_cast<float*>(wsp) : nullptr;
    p.stages = pl.stages; p.a_bytes = pl.a_bytes; p.b_bytes = pl.b_bytes;
    p.stage_bytes = pl.stage_bytes; p.acc_stride = pl.acc_stride;
    p.a_e = a_e; p.b_e = a_e;
    p.prog = prog;
    p.pace = pl.kb_per_split >= kPaceMinKb ? kPaceKb : 0;
    if (p.pace) SKP_CUDA(cudaMemsetAsync(prog, 0, kPaceBytes, st));
    // the Gram of rows (kmajor) decides the final basis' orthonormality and
    // feeds the error identity: 256-deep promotion chains there (its tiles
    // are few and short, so the extra epilogue drains are hidden)
    p.chunk_kb = kmajor ? 4 : h_chunk_kb();
    p.emit_hi = nullptr; p.emit_lo = nullptr; p.emit_e = nullptr; p.overflow = nullptr;
    // kind::f16: D f32, A and B f16, both MN-major (bits 15, 16) or both K-major
    const uint32_t mn = kmajor ? 0u : 1u;
    p.idesc = (1u << 4) | (mn << 15) | (mn << 16) | ((uint32_t)(p.bn >> 3) << 17) |
              ((uint32_t)(sp.R >> 4) << 24);
    CUtensorMap mah, mal, mbh, mbl;
    bool ok;
    if (kmajor)
        ok = h_encode_k(&mah, Ahi, (uint64_t)K, (uint64_t)N, lda, HM) &&
             h_encode_k(&mal, Alo, (uint64_t)K, (uint64_t)N, lda, HM) &&
             h_encode_k(&mbh, Ahi, (uint64_t)K, (uint64_t)N, lda, (uint32_t)sp.bcols) &&
             h_encode_k(&mbl, Alo, (uint64_t)K, (uint64_t)N, lda, (uint32_t)sp.bcols);
    else
        ok = h_encode_mn(&mah, Ahi, (uint64_t)N, (uint64_t)K, lda) &&
             h_encode_mn(&mal, Alo, (uint64_t)N, (uint64_t)K, lda) &&
             h_encode_mn(&mbh, Ahi, (uint64_t)N, (uint64_t)K, lda, (uint32_t)sp.bcols) &&
             h_encode_mn(&mbl, Alo, (uint64_t)N, (uint64_t)K, lda, (uint32_t)sp.bcols);
    if (!ok) {
        set_error("cuTensorMapEncodeTiled failed (syrk_h3)");
        return SKP_ERR_UNSUPPORTED;
    }
    const int units = p.sym;
    if (pair) {
        SKP_CUDA(cudaFuncSetAttribute(gemm_h3_kernel<true, 6>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(2 * std::min(units, h_sms / 2)));
        cfg.blockDim = dim3(kHThreads);
        cfg.dynamicSmemBytes = pl.smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        SKP_CUDA(cudaLaunchKernelEx(&cfg, gemm_h3_kernel<true, 6>, mah, mal, mbh, mbl, p));
        SKP_LAUNCHED(gemm_h3_kernel_pair);
    } else {
        SKP_CUDA(cudaFuncSetAttribute(gemm_h3_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
        gemm_h3_kernel<false><<<std::min(units, h_sms), kHThreads, pl.smem, st>>>(mah, mal, mbh, mbl,
                                                                                 p);
        SKP_LAUNCHED(gemm_h3_kernel);
    }
    if (splits > 1) {
        const int64_t blocks = std::min<int64_t>(cdiv(N * N, 256), (int64_t)h_sms * 8);
        h3_splitk_reduce<<<(unsigned)blocks, 256, 0, st>>>(p.ws, splits, N, N, alpha, beta, C, ldc);
        SKP_LAUNCHED(h3_splitk_reduce);
    }
    const unsigned nt = (unsigned)cdiv(N, 32);
    sym_mirror_kernel<<<dim3(nt, nt), dim3(32, 8), 0, st>>>(C, N, ldc);
    SKP_LAUNCHED(sym_mirror_kernel);
    return SKP_OK;
}

int gemm_h3(int ta, int64_t M, int64_t N, int64_t K, float alpha, const void* Ahi, const void* Alo,
            int64_t lda, const int32_t* a_e, const void* Bhi, const void* Blo, int64_t ldb,
            const int32_t* b_e, float beta, float* C, int64_t ldc, void* ws, int64_t ws_bytes,
            cudaStream_t st) {
    return gemm_h3_impl(ta, M, N, K, alpha, Ahi, Alo, lda, a_e, Bhi, Blo, ldb, b_e, beta, C, ldc,
                        ws, ws_bytes, nullptr, st);
}

int64_t gemm_h3s_ws_bytes(int64_t M, int64_t N, int64_t K) {
    if (!h_init()) return 0;
    const HPlan pl = hs_plan(M, N, K, INT64_MAX, h_pair(M));
    return kPaceBytes + (pl.splits > 1 ? (int64_t)pl.splits * M * N * 4 : 0);
}

int gemm_h3s(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
             const int32_t* a_e, const void* Bhi, const void* Blo, int64_t ldb, const int32_t* b_e,
             float beta, float* C, int64_t ldc, int32_t* overflow, void* ws, int64_t ws_bytes,
             cudaStream_t st) {
    if (!h_init()) {
        set_error("unsupported: the 3xFP16 tcgen05 GEMM needs an sm_100 device");
        return SKP_ERR_UNSUPPORTED;
    }
    if (M == 0 || N == 0) return SKP_OK;
    if (K == 0 || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) {
        set_error("unsupported: gemm_h3s sizes");
        return SKP_ERR_UNSUPPORTED;
    }
    const uintptr_t al = reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(Bhi) |
                         reinterpret_cast<uintptr_t>(Blo);
    if ((al & 15) || (lda & 31) || (ldb & 7)) {
        set_error("unsupported: gemm_h3s needs 16-byte aligned operands, lda %% 32 == 0, "
                  "ldb %% 8 == 0 (lda=%lld ldb=%lld)", (long long)lda, (long long)ldb);
        return SKP_ERR_UNSUPPORTED;
    }
    const bool pair = h_pair(M);
    // ws: [pacing slots | split-K partials]
    unsigned* prog = (ws && ws_bytes >= kPaceBytes) ? reinterpret_cast<unsigned*>(ws) : nullptr;
    void* wsp = prog ? reinterpret_cast<char*>(ws) + kPaceBytes : ws;
    const int64_t wsp_bytes = prog ? ws_bytes - kPaceBytes : ws_bytes;
    const int64_t cap = wsp ? wsp_bytes / 4 : 0;
    HPlan pl = hs_plan(M, N, K, cap, pair);
    if (pl.splits > 1 && (!wsp || (int64_t)pl.splits * M * N * 4 > wsp_bytes))
        pl = hs_plan(M, N, K, 0, pair);
    H3SParams p;
    p.M = (int)M; p.N = (int)N; p.K = (int)K;
    p.bn = pl.bn; p.tiles_m = pl.tiles_m; p.tiles_n = pl.tiles_n; p.splits = pl.splits;
    p.kb_per_split = pl.kb_per_split; p.num_kb = pl.num_kb;
    p.alpha = alpha; p.beta = beta; p.C = C; p.ldc = ldc;
    p.ws = pl.splits > 1 ? reinterpret_cast<float*>(wsp) : nullptr;
    p.stages = pl.stages; p.a_bytes = pl.a_bytes; p.b_bytes = pl.b_bytes;
    p.stage_bytes = pl.stage_bytes; p.acc_stride = pl.acc_stride;
    p.a_e = a_e; p.b_e = b_e; p.overflow = overflow;
    p.prog = prog;
    p.pace = (prog && pl.kb_per_split >= kPaceMinKb) ? kPaceKbS : 0;
    if (p.pace) SKP_CUDA(cudaMemsetAsync(prog, 0, kPaceBytes, st));
    p.chunk_kb = h_chunk_kb();
    if (2 * p.acc_stride + kSSlots * (int)kSSlotCols > (int)kHTmemCols || p.bn > kSMaxBn) {
        set_error("internal: gemm_h3s tile does not fit TMEM (bn=%d)", p.bn);
        return SKP_ERR_UNSUPPORTED;
    }
    // A from TMEM (K-major there), B K-major
    p.idesc = (1u << 4) | ((uint32_t)(p.bn >> 3) << 17) |
              ((uint32_t)((pair ? 2 * HM : HM) >> 4) << 24);
    CUtensorMap ma, mbh, mbl;
    const int bcols = pair ? p.bn / 2 : p.bn;
    const bool ok = hs_encode_a(&ma, A, (uint64_t)M, (uint64_t)K, lda) &&
                    h_encode_k(&mbh, Bhi, (uint64_t)K, (uint64_t)N, ldb, (uint32_t)bcols) &&
                    h_encode_k(&mbl, Blo, (uint64_t)K, (uint64_t)N, ldb, (uint32_t)bcols);
    if (!ok) {
        set_error("cuTensorMapEncodeTiled failed (gemm_h3s)");
        return SKP_ERR_UNSUPPORTED;
    }
    const int units = p.tiles_m * p.tiles_n * p.splits;
    if (pair) {
        SKP_CUDA(cudaFuncSetAttribute(gemm_h3s_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(2 * std::min(units, h_sms / 2)));
        cfg.blockDim = dim3(kSThreads);
        cfg.dynamicSmemBytes = pl.smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        SKP_CUDA(cudaLaunchKernelEx(&cfg, gemm_h3s_kernel<true>, ma, mbh, mbl, p));
        SKP_LAUNCHED(gemm_h3s_kernel_pair);
    } else {
        SKP_CUDA(cudaFuncSetAttribute(gemm_h3s_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
        gemm_h3s_kernel<false><<<std::min(units, h_sms), kSThreads, pl.smem, st>>>(ma, mbh, mbl, p);
        SKP_LAUNCHED(gemm_h3s_kernel);
    }
    if (p.splits > 1) {
        const int64_t blocks = std::min<int64_t>(cdiv(M * N, 256), (int64_t)h_sms * 8);
        h3_splitk_reduce<<<(unsigned)blocks, 256, 0, st>>>(p.ws, p.splits, M, N, alpha, beta, C,
                                                           ldc);
        SKP_LAUNCHED(h3_splitk_reduce);
    }
    return SKP_OK;
}

int h2_exponent(const float* X, int64_t rows, int64_t cols, int64_t ld, int32_t* e_io,
                int have_amax, int margin, cudaStream_t st) {
    uint32_t* amax = reinterpret_cast<uint32_t*>(e_io + 1);
    if (!have_amax) {
        SKP_CUDA(cudaMemsetAsync(amax, 0, 4, st));
        if (rows > 0 && cols > 0) {
            const int64_t work = rows * cdiv(cols, 4);
            const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(work, 256), (int64_t)h_sms * 16);
            absmax_kernel<<<blocks, 256, 0, st>>>(X, rows, cols, ld, amax);
            SKP_LAUNCHED(absmax_kernel);
        }
    }
    h2_exponent_kernel<<<1, 32, 0, st>>>(e_io, margin);
    SKP_LAUNCHED(h2_exponent_kernel);
    return SKP_OK;
}

int split_h2_inplace(float* X, int64_t rows, int64_t cols, int64_t ld, int32_t* e,
                     int have_amax, cudaStream_t st) {
    if (rows == 0 || cols == 0) {
        SKP_CUDA(cudaMemsetAsync(e, 0, 4, st));
        return SKP_OK;
    }
    SKP_ARG((ld & 7) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 && cols <= ld,
            "split_h2_inplace: needs 16-byte aligned rows with ld %% 8 == 0");
    SKP_ARG(cols * 4 <= 200 * 1024, "split_h2_inplace: row too long for shared memory");
    uint32_t* amax = reinterpret_cast<uint32_t*>(e + 1);
    if (!have_amax) {
        SKP_CUDA(cudaMemsetAsync(amax, 0, 4, st));
        const int64_t work = rows * cdiv(cols, 4);
        const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(work, 256), (int64_t)h_sms * 16);
        absmax_kernel<<<blocks, 256, 0, st>>>(X, rows, cols, ld, amax);
        SKP_LAUNCHED(absmax_kernel);
    }
    const size_t smem = (size_t)cols * 4;
    SKP_CUDA(cudaFuncSetAttribute(split_h2_inplace_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned blocks = (unsigned)std::min<int64_t>(rows, (int64_t)h_sms * 16);
    split_h2_inplace_kernel<<<blocks, 256, smem, st>>>(X, rows, cols, ld, amax, e);
    SKP_LAUNCHED(split_h2_inplace_kernel);
    return SKP_OK;
}

int split_h2(const float* X, int64_t rows, int64_t cols, int64_t ld, int trans, void* hi, void* lo,
             int64_t ldh, int32_t* e, int have_amax, cudaStream_t st) {
    if (rows == 0 || cols == 0) {
        SKP_CUDA(cudaMemsetAsync(e, 0, 4, st));
        return SKP_OK;
    }
    uint32_t* amax = reinterpret_cast<uint32_t*>(e + 1);
    const int64_t work = rows * cdiv(cols, 4);
    const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(work, 256), (int64_t)h_sms * 16);
    if (!have_amax) {
        SKP_CUDA(cudaMemsetAsync(amax, 0, 4, st));
        absmax_kernel<<<blocks, 256, 0, st>>>(X, rows, cols, ld, amax);
        SKP_LAUNCHED(absmax_kernel);
    }
    if (!trans) {
        split_h2_kernel<<<blocks, 256, 0, st>>>(X, rows, cols, ld, amax, (__half*)hi, (__half*)lo,
                                                ldh, e);
        SKP_LAUNCHED(split_h2_kernel);
    } else {
        SKP_ARG(cdiv(rows, 64) <= 65535, "split_h2: too many rows for the transposing split");
        split_h2_t_kernel<<<dim3((unsigned)cdiv(cols, 64), (unsigned)cdiv(rows, 64)), 256, 0, st>>>(
            X, rows, cols, ld, amax, (__half*)hi, (__half*)lo, ldh, e);
        SKP_LAUNCHED(split_h2_t_kernel);
    }
    return SKP_OK;
}

}  // namespace skp

using namespace skp;

extern "C" int64_t skp_gemm_h3_ws_bytes(int transA, int64_t M, int64_t N, int64_t K) {
    return gemm_h3_ws_bytes(transA, M, N, K);
}

extern "C" int skp_gemm_h3(int transA, int64_t M, int64_t N, int64_t K, float alpha,
                           const void* A_hi, const void* A_lo, int64_t lda, const int32_t* a_exp,
                           const void* B_hi, const void* B_lo, int64_t ldb, const int32_t* b_exp,
                           float beta, float* C, int64_t ldc, void* ws, int64_t ws_bytes,
                           void* stream) {
    SKP_ARG(M >= 0 && N >= 0 && K >= 0, "gemm_h3: negative size");
    SKP_ARG(transA == 0 || transA == 1, "gemm_h3: transA must be 0/1");
    SKP_ARG(lda >= (transA ? M : K) && lda >= 1, "gemm_h3: lda too small");
    SKP_ARG(ldb >= K && ldb >= 1, "gemm_h3: ldb too small");
    SKP_ARG(ldc >= N && ldc >= 1, "gemm_h3: ldc too small");
    SKP_ARG((M == 0 || N == 0 || K == 0 || (A_hi && A_lo && B_hi && a_exp && b_exp)) &&
                (M == 0 || N == 0 || C),
            "gemm_h3: null pointer");
    return gemm_h3(transA, M, N, K, alpha, A_hi, A_lo, lda, a_exp, B_hi, B_lo, ldb, b_exp, beta, C,
                   ldc, ws, ws_bytes, SKP_STREAM(stream));
}

extern "C" int skp_split_h2_f32(const float* X, int64_t rows, int64_t cols, int64_t ld,
                                int32_t trans, void* hi, void* lo, int64_t ldh, int32_t* e,
                                int32_t have_amax, void* stream) {
    SKP_ARG(rows >= 0 && cols >= 0 && ld >= cols && ld >= 1, "split_h2: bad sizes");
    SKP_ARG(trans == 0 || trans == 1, "split_h2: trans must be 0/1");
    SKP_ARG(ldh >= (trans ? rows : cols), "split_h2: ldh too small");
    SKP_ARG(e && (rows == 0 || cols == 0 || (X && hi && lo)), "split_h2: null pointer");
    h_init();
    return split_h2(X, rows, cols, ld, trans, hi, lo, ldh, e, have_amax != 0, SKP_STREAM(stream));
}

extern "C" int64_t skp_syrk_h3_ws_bytes(int64_t N, int64_t K) { return skp::syrk_h3_ws_bytes(N, K); }

extern "C" int skp_syrk_h3(int32_t kmajor, int64_t N, int64_t K, float alpha, const void* A_hi,
                           const void* A_lo, int64_t lda, const int32_t* a_exp, float beta,
                           float* C, int64_t ldc, void* ws, int64_t ws_bytes, void* stream) {
    SKP_ARG(N >= 0 && K >= 0 && lda >= (kmajor ? K : N) && ldc >= N && a_exp &&
                (N == 0 || (A_hi && A_lo && C)),
            "syrk_h3: bad arguments");
    return skp::syrk_h3(kmajor, N, K, alpha, A_hi, A_lo, lda, a_exp, beta, C, ldc, ws, ws_bytes,
                        SKP_STREAM(stream));
}

extern "C" int64_t skp_gemm_h3s_ws_bytes(int64_t M, int64_t N, int64_t K) {
    return gemm_h3s_ws_bytes(M, N, K);
}

extern "C" int skp_gemm_h3s(int64_t M, int64_t N, int64_t K, float alpha, const float* A,
                            int64_t lda, const int32_t* a_exp, const void* B_hi, const void* B_lo,
                            int64_t ldb, const int32_t* b_exp, float beta, float* C, int64_t ldc,
                            int32_t* overflow, void* ws, int64_t ws_bytes, void* stream) {
    SKP_ARG(M >= 0 && N >= 0 && K >= 0, "gemm_h3s: negative size");
    SKP_ARG(lda >= M && lda >= 1, "gemm_h3s: lda too small");
    SKP_ARG(ldb >= K && ldb >= 1, "gemm_h3s: ldb too small");
    SKP_ARG(ldc >= N && ldc >= 1, "gemm_h3s: ldc too small");
    SKP_ARG((M == 0 || N == 0 || K == 0 || (A && B_hi && B_lo && a_exp && b_exp)) &&
                (M == 0 || N == 0 || C),
            "gemm_h3s: null pointer");
    return gemm_h3s(M, N, K, alpha, A, lda, a_exp, B_hi, B_lo, ldb, b_exp, beta, C, ldc, overflow,
                    ws, ws_bytes, SKP_STREAM(stream));
}

extern "C" int skp_h2_exponent_f32(const float* X, int64_t rows, int64_t cols, int64_t ld,
                                   int32_t* e_io, int32_t have_amax, int32_t margin_bits,
                                   void* stream) {
    SKP_ARG(rows >= 0 && cols >= 0 && ld >= cols && e_io, "h2_exponent: bad arguments");
    SKP_ARG(margin_bits >= 0 && margin_bits <= 60, "h2_exponent: margin_bits out of range");
    h_init();
    return h2_exponent(X, rows, cols, ld, e_io, have_amax != 0, margin_bits, SKP_STREAM(stream));
}

extern "C" int skp_gemm_h3_emit_t(int transA, int64_t M, int64_t N, int64_t K, float alpha,
                                  const void* A_hi, const void* A_lo, int64_t lda,
                                  const int32_t* a_exp, const void* B_hi, const void* B_lo,
                                  int64_t ldb, const int32_t* b_exp, void* Ct_hi, void* Ct_lo,
                                  int64_t ldct, int32_t shift, int32_t fixed, int32_t e_fixed,
                                  int32_t* e_out, int32_t* overflow, int32_t b_lower, void* ws,
                                  int64_t ws_bytes, void* stream) {
    SKP_ARG(M >= 0 && N >= 0 && K >= 0, "gemm_h3_emit_t: negative size");
    SKP_ARG(transA == 0 || transA == 1, "gemm_h3_emit_t: transA must be 0/1");
    SKP_ARG(lda >= (transA ? M : K) && lda >= 1, "gemm_h3_emit_t: lda too small");
    SKP_ARG(ldb >= K && ldb >= 1, "gemm_h3_emit_t: ldb too small");
    SKP_ARG(ldct >= M, "gemm_h3_emit_t: ldct too small");
    SKP_ARG(Ct_hi && Ct_lo && e_out && A_hi && A_lo && B_hi && a_exp && b_exp,
            "gemm_h3_emit_t: null pointer");
    H3Emit em{Ct_hi, Ct_lo, ldct, shift, fixed, e_fixed, e_out, overflow, b_lower ? 1 : 0};
    return gemm_h3_impl(transA, M, N, K, alpha, A_hi, A_lo, lda, a_exp, B_hi, B_lo, ldb, b_exp,
                        0.f, nullptr, 0, ws, ws_bytes, &em, SKP_STREAM(stream));
}

extern "C" int skp_split_h2_inplace_f32(float* X, int64_t rows, int64_t cols, int64_t ld,
                                        int32_t* e, int32_t have_amax, void* stream) {
    SKP_ARG(rows >= 0 && cols >= 0 && ld >= cols && ld >= 1 && e && (rows == 0 || cols == 0 || X),
            "split_h2_inplace: bad arguments");
    h_init();
    return split_h2_inplace(X, rows, cols, ld, e, have_amax != 0, SKP_STREAM(stream));
}
