// K2 v1: A~ = A . S with 32 rows of A in the 32 lanes of every warp.
//
// Why this shape: every A element must reach s = 8 random output columns.
// With lane = row, all 32 lanes of a warp need the SAME A column j at the
// same time (the sketch structure is shared by all rows), so the gather
// A_s[j][lane] is one conflict-free shared-memory wavefront, and the sign /
// column metadata is a warp-uniform broadcast.  Output accumulators live in
// registers: warp w owns CW output columns for its 32 rows.
//
//   grid  : (ceil(m/32) row blocks) x (P column slices), slice index fastest,
//           so the P CTAs of one row block run together and share the block
//           through L2 (one HBM read of A).  Slice = 16 warps x CW columns.
//   chunk : A is streamed in column chunks of J (32 rows x J, transposed into
//           smem with a 33-word row pitch -> conflict-free on both sides);
//           chunk k+1 is prefetched into registers while chunk k is reduced;
//           its metadata arrives by cp.async into a double buffer.
//   meta  : padded-ELL view of S per chunk: for chunk k and column c one
//           16-byte record {slot0, slot1, slot2, overflow}; slots are smem
//           BYTE offsets into [+A chunk | -A chunk | zero row] (the chunk is
//           stored twice, negated copy second, so the sign is the offset);
//           unused slots point at the zero row; overflow packs the chunk-local
//           start (low 16 bits) and count (high 16) of the rare >3-entry tail,
//           staged per chunk in smem.  With J*s/l ~ 1 entry per (chunk, column)
//           a column costs ~11 instructions with one rarely-taken branch, and
//           consecutive columns are independent (ILP).  The ELL is padded to
//           whole slices, so the column sweep has no bounds checks.
//   out   : per-warp tiles transposed through smem -> coalesced row stores.
// ||A||_F^2 and the non-finite count are fused into slice 0's loads.
#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace skp {
namespace {

constexpr int kRowsNW = 16;                  // warps per CTA
constexpr int kRowsThreads = 32 * kRowsNW;
constexpr int kPitch = 33;                   // smem words per A column (32 rows + 1)

template <typename T>
struct RowsCfg;
template <>
struct RowsCfg<float> {
    static constexpr int J = 512, CW = 64, VEC = 4;
};
template <>
struct RowsCfg<double> {
    static constexpr int J = 256, CW = 32, VEC = 2;
};

__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

template <typename T, typename V>
__device__ __noinline__ V load_tail(const T* A, int64_t lda, int64_t m, int64_t n, int64_t row,
                                    int64_t col) {
    T t[sizeof(V) / sizeof(T)];
#pragma unroll
    for (int e = 0; e < (int)(sizeof(V) / sizeof(T)); ++e)
        t[e] = (row < m && col + e < n) ? A[row * lda + col + e] : T(0);
    return *reinterpret_cast<V*>(t);
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
template <typename T>
__device__ __forceinline__ T lds_t(uint32_t a);
template <>
__device__ __forceinline__ float lds_t<float>(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
template <>
__device__ __forceinline__ double lds_t<double>(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

// smem layout: As[2J+1][kPitch] T (+A | -A | zero row) | ell[2][SW] int4 |
//              ovf[2][J*8] int | chunk overflow bounds [nchunks+1] int | red
template <typename T>
struct RowsSmem {
    static constexpr int J = RowsCfg<T>::J, CW = RowsCfg<T>::CW;
    static constexpr int SW = kRowsNW * CW;
    static constexpr size_t chunk_bytes = (size_t)(2 * J + 1) * kPitch * sizeof(T);
    static constexpr size_t tile_bytes = (size_t)kRowsNW * 32 * (CW + 1) * sizeof(T);
    static constexpr size_t as_bytes =
        ((chunk_bytes > tile_bytes ? chunk_bytes : tile_bytes) + 15) / 16 * 16;
    static constexpr int OVMAX = J * 8;  // a chunk holds J*s entries; overflow <= that (s <= 8)
    static constexpr int MAXCH = 512;    // chunks staged (n <= 512 * J)
    static constexpr size_t bytes =
        as_bytes + 2 * (size_t)SW * 16 + 2 * (size_t)OVMAX * 4 + (MAXCH + 1) * 4 + 64 * 8;
    static constexpr uint32_t zero_off = (uint32_t)(2 * J * kPitch * sizeof(T));
};

template <typename T>
__global__ void __launch_bounds__(kRowsThreads, 1)
sketch_rows_kernel(const T* __restrict__ A, int64_t lda, int64_t m, int64_t n, int nchunks,
                   int P, const int4* __restrict__ ell, const int32_t* __restrict__ ovf,
                   const int32_t* __restrict__ optr, int64_t rpad,
                   int64_t r, T scale, T* __restrict__ out, int64_t ldo, double* fro2,
                   long long* nonfinite) {
    using C = RowsSmem<T>;
    constexpr int J = C::J, CW = C::CW, SW = C::SW, VEC = RowsCfg<T>::VEC;
    constexpr int TC = 8 * VEC;                       // tile cols per warp load (4 rows x TC)
    constexpr int NT = (32 / 4) * (J / TC);           // tiles per chunk
    constexpr int PER = NT / kRowsNW;                 // tiles per warp
    static_assert(NT % kRowsNW == 0, "tile split");
    typedef typename std::conditional<sizeof(T) == 4, float4, double2>::type V;

    extern __shared__ __align__(16) unsigned char sm[];
    T* As = reinterpret_cast<T*>(sm);
    int4* ell_s = reinterpret_cast<int4*>(sm + C::as_bytes);
    int32_t* ovf_s = reinterpret_cast<int32_t*>(ell_s + 2 * SW);
    int32_t* cbound = ovf_s + 2 * C::OVMAX;       // overflow index range of chunk k
    double* red_d = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(cbound + C::MAXCH + 1) + 15) & ~uintptr_t(15));
    long long* red_i = reinterpret_cast<long long*>(red_d + 32);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t rb = blockIdx.x / P;
    const int slice = blockIdx.x % P;
    const int64_t i0 = rb * 32;
    const int64_t c0 = (int64_t)slice * SW;
    const int64_t c1 = c0 + SW < r ? c0 + SW : r;        // slice columns [c0, c1)
    const bool count_norms = slice == 0 && (fro2 || nonfinite);

    // ---- ELL records of chunk k for this slice -> ell_s[b] (cp.async 16 B) ----
    auto load_meta = [&](int k, int b) {
        const int4* src = ell + (int64_t)k * rpad + c0;
        int4* dst = ell_s + b * SW;
        const int nrec = SW;
        for (int i = threadIdx.x; i < nrec; i += kRowsThreads)
            cp_async16((uint32_t)__cvta_generic_to_shared(dst + i), src + i);
        // the whole chunk's overflow block (all columns; ~J*s*P(cnt>2)/... ints)
        const int ob = cbound[k], oe = cbound[k + 1];
        const int no = oe - ob < C::OVMAX ? oe - ob : C::OVMAX;
        int32_t* od = ovf_s + b * C::OVMAX;
        for (int i = threadIdx.x; i < no; i += kRowsThreads)
            cp_async4((uint32_t)__cvta_generic_to_shared(od + i), ovf + ob + i);
    };

    // ---- A chunk prefetch (registers) and transposed store ---------------------
    V pre[PER];
    double ss = 0.0;
    long long bad = 0;
    auto prefetch = [&](int k) {
        const int64_t j0 = (int64_t)k * J;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int tile = warp + kRowsNW * q;
            const int trow = tile % 8, tcol = tile / 8;
            const int64_t row = i0 + trow * 4 + (lane >> 3);
            const int64_t col = j0 + (int64_t)tcol * TC + (lane & 7) * VEC;
            V v;
            if (row < m && col + VEC <= n) {
                v = __ldg(reinterpret_cast<const V*>(A + row * lda + col));
            } else {
                v = load_tail<T, V>(A, lda, m, n, row, col);
            }
            pre[q] = v;
            if (count_norms) {
                const T* t = reinterpret_cast<const T*>(&v);
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    ss += (double)t[e] * (double)t[e];
                    bad += !isfinite(t[e]);
                }
            }
        }
    };
    auto store_chunk = [&]() {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int tile = warp + kRowsNW * q;
            const int trow = tile % 8, tcol = tile / 8;
            const int rloc = trow * 4 + (lane >> 3);
            const int jloc = tcol * TC + (lane & 7) * VEC;
            const T* t = reinterpret_cast<const T*>(&pre[q]);
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                As[(jloc + e) * kPitch + rloc] = t[e];
                As[(J + jloc + e) * kPitch + rloc] = -t[e];
            }
        }
    };

    T acc[CW];
#pragma unroll
    for (int i = 0; i < CW; ++i) acc[i] = T(0);

    // zero row (target of unused ELL slots) and chunk overflow bounds, once
    for (int i = threadIdx.x; i < kPitch; i += kRowsThreads) As[2 * J * kPitch + i] = T(0);
    for (int i = threadIdx.x; i <= nchunks; i += kRowsThreads) cbound[i] = __ldg(optr + (int64_t)i * r);
    __syncthreads();
    load_meta(0, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    prefetch(0);
    const uint32_t x_base = (uint32_t)__cvta_generic_to_shared(As) + lane * (uint32_t)sizeof(T);
    const int cl0 = warp * CW;
    (void)cl0;
    for (int k = 0; k < nchunks; ++k) {
        const int b = k & 1;
        store_chunk();
        cp_async_wait_all();
        __syncthreads();
        if (k + 1 < nchunks) {
            load_meta(k + 1, b ^ 1);
            asm volatile("cp.async.commit_group;" ::: "memory");
            prefetch(k + 1);
        }
        const int4* rec = ell_s + b * SW + cl0;
        const int32_t* ovk = ovf_s + b * C::OVMAX;
        // columns in batches of KB: all record loads, then all slot loads, no
        // per-column branch (ILP across columns); unused slots (zero row) are
        // predicated off so they cost no shared-memory wavefront; the rare
        // >3-entry overflow is one warp-uniform check per batch
        constexpr int KB = 4;
        const int zo = (int)C::zero_off;
#pragma unroll
        for (int kb0 = 0; kb0 < CW; kb0 += KB) {
            int4 d[KB];
#pragma unroll
            for (int i = 0; i < KB; ++i) d[i] = rec[kb0 + i];
            int ovf_any = 0;
#pragma unroll
            for (int i = 0; i < KB; ++i) {
                T a = T(0);
                if (d[i].x != zo) a += lds_t<T>(x_base + (uint32_t)d[i].x);
                if (d[i].y != zo) a += lds_t<T>(x_base + (uint32_t)d[i].y);
                if (d[i].z != zo) a += lds_t<T>(x_base + (uint32_t)d[i].z);
                acc[kb0 + i] += a;
                ovf_any |= d[i].w;
            }
            if (ovf_any) {
#pragma unroll
                for (int i = 0; i < KB; ++i) {
                    if (d[i].w) {
                        const int o = d[i].w & 0xffff, e = o + (d[i].w >> 16);
                        T a = T(0);
#pragma unroll 1
                        for (int t = o; t < e; ++t) a += lds_t<T>(x_base + (uint32_t)ovk[t]);
                        acc[kb0 + i] += a;
                    }
                }
            }
        }
        __syncthreads();
    }

    // ---- fused norms ---------------------------------------------------------
    if (count_norms) {
        double bs = block_sum<double>(ss, red_d);
        long long bb = block_sum<long long>(bad, red_i);
        if (threadIdx.x == 0) {
            if (fro2) atomicAdd(fro2, bs);
            if (nonfinite && bb) atomicAdd((unsigned long long*)nonfinite, (unsigned long long)bb);
        }
    }

    // ---- output: per-warp [32 rows x CW] tile through smem, coalesced rows ----
    T* tile = As + warp * (32 * (CW + 1));
#pragma unroll
    for (int kc = 0; kc < CW; ++kc) tile[lane * (CW + 1) + kc] = acc[kc] * scale;
    __syncwarp();
    const int64_t cbase = c0 + warp * CW;
    for (int rr = 0; rr < 32; ++rr) {
        const int64_t row = i0 + rr;
        if (row >= m) break;
        for (int kc = lane; kc < CW; kc += 32) {
            const int64_t col = cbase + kc;
            if (col < c1) out[row * ldo + col] = tile[rr * (CW + 1) + kc];
        }
    }
}

// ---- padded-ELL build (per sketch, per chunk width J) -------------------------
// ovf_cnt[k*r + c] = max(0, #entries of column c in chunk k - 3)
__global__ void ell_count_kernel(const int32_t* __restrict__ colptr,
                                 const int32_t* __restrict__ entries, int64_t r, int J,
                                 int32_t* __restrict__ ovf_cnt) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < r;
         c += (int64_t)gridDim.x * blockDim.x) {
        int prev_k = -1, run = 0;
        for (int e = colptr[c]; e <= colptr[c + 1]; ++e) {   // entries ascending in j
            int k = e < colptr[c + 1] ? (int)((((uint32_t)entries[e]) & 0x7fffffffu) / (uint32_t)J)
                                      : -2;
            if (k != prev_k) {
                if (prev_k >= 0 && run > 3) ovf_cnt[(int64_t)prev_k * r + c] = run - 3;
                prev_k = k;
                run = 0;
            }
            ++run;
        }
    }
}

// multi-block exclusive scan (in place), 3 phases
constexpr int kScanB = 1024;
__global__ void scan_block_sums(const int32_t* __restrict__ x, int64_t n,
                                int64_t* __restrict__ sums) {
    __shared__ long long red[32];
    long long s = 0;
    const int64_t b0 = (int64_t)blockIdx.x * kScanB * 8;
    for (int64_t i = b0 + threadIdx.x; i < b0 + kScanB * 8 && i < n; i += kScanB) s += x[i];
    s = block_sum<long long>(s, red);
    if (threadIdx.x == 0) sums[blockIdx.x] = s;
}
__global__ void scan_sums_serial(int64_t* sums, int64_t nb, int32_t* total_out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int64_t acc = 0;
        for (int64_t i = 0; i < nb; ++i) {
            int64_t v = sums[i];
            sums[i] = acc;
            acc += v;
        }
        *total_out = (int32_t)acc;
    }
}
__global__ void scan_apply(int32_t* x, int64_t n, const int64_t* __restrict__ sums) {
    __shared__ long long buf[kScanB];
    const int64_t b0 = (int64_t)blockIdx.x * kScanB * 8;
    long long carry = sums[blockIdx.x];
    for (int part = 0; part < 8; ++part) {
        const int64_t i = b0 + (int64_t)part * kScanB + threadIdx.x;
        long long v = i < n ? x[i] : 0;
        buf[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < kScanB; o <<= 1) {
            long long t = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
            __syncthreads();
            buf[threadIdx.x] += t;
            __syncthreads();
        }
        if (i < n) x[i] = (int32_t)(carry + buf[threadIdx.x] - v);
        long long tot = buf[kScanB - 1];
        __syncthreads();
        carry += tot;
    }
}

// ell[k*rpad + c] = {slot0, slot1, slot2, overflow}; columns r..rpad-1 are
// all-zero-row padding.  Overflow start is chunk-local (ovf index - ovf_ptr[k*r]).
__global__ void ell_fill_kernel(const int32_t* __restrict__ colptr,
                                const int32_t* __restrict__ entries, int64_t r, int64_t rpad,
                                int J, int nchunks, int elem, uint32_t zero_off,
                                const int32_t* __restrict__ ovf_ptr, int4* __restrict__ ell,
                                int32_t* __restrict__ ovf) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < rpad;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int z = (int)zero_off;
        if (c >= r) {
            for (int k = 0; k < nchunks; ++k) ell[(int64_t)k * rpad + c] = make_int4(z, z, z, 0);
            continue;
        }
        int e = colptr[c];
        const int e1 = colptr[c + 1];
        for (int k = 0; k < nchunks; ++k) {
            int slot[3] = {z, z, z};
            int o = ovf_ptr[(int64_t)k * r + c], i = 0;
            const int o0 = o, cbase = ovf_ptr[(int64_t)k * r];
            for (; e < e1; ++e, ++i) {
                const uint32_t v = (uint32_t)entries[e];
                const uint32_t j = v & 0x7fffffffu;
                if ((int)(j / (uint32_t)J) != k) break;
                const uint32_t jl = (j - (uint32_t)k * J) + ((v >> 31) ? (uint32_t)J : 0u);
                const int off = (int)(jl * kPitch * elem);
                if (i < 3) slot[i] = off;
                else ovf[o++] = off;
            }
            const int cnt = o - o0;
            ell[(int64_t)k * rpad + c] =
                make_int4(slot[0], slot[1], slot[2], cnt ? ((o0 - cbase) | (cnt << 16)) : 0);
        }
    }
}

}  // namespace

// workspace: ell (nch*r int4) | ovf_cnt/ptr (nch*r+1 int) | ovf (n*s int) | scan sums
int64_t rows_chunk_ws(int64_t n, int32_t s, int64_t r, int J, int SW) {
    int64_t nch = cdiv(n, J);
    int64_t rpad = cdiv(r, SW) * SW;
    int64_t slots = nch * r + 1;
    int64_t nb = cdiv(slots, kScanB * 8);
    return nch * rpad * 16 + slots * 4 + n * s * 4 + nb * 8 + 256;
}

template <typename T>
int sketch_right_rows(const T* A, int64_t lda, int64_t m, int64_t n, const int32_t* colptr,
                      const int32_t* entries, int32_t s, int64_t r, T* out, int64_t ldo,
                      double* fro2, int64_t* nonfinite, void* ws, int64_t ws_bytes,
                      cudaStream_t st) {
    using C = RowsSmem<T>;
    constexpr int J = C::J;
    const int64_t nch = cdiv(n, J);
    const int64_t slots = nch * r + 1;
    const int64_t rpad = cdiv(r, C::SW) * C::SW;
    if (ws_bytes < rows_chunk_ws(n, s, r, J, C::SW)) return SKP_ERR_UNSUPPORTED;
    // chunk-local overflow offsets are packed in 16 bits
    if (J * s >= 65536) return SKP_ERR_UNSUPPORTED;
    if ((reinterpret_cast<uintptr_t>(A) & 15) || ((lda * (int64_t)sizeof(T)) & 15))
        return SKP_ERR_UNSUPPORTED;
    // staged overflow block per chunk <= J*s entries; chunk bounds staged in smem
    if (s > 8 || nch > C::MAXCH || n * s >= 0x7fffffffLL || slots >= 0x7fffffffLL)
        return SKP_ERR_UNSUPPORTED;
    int4* ell = reinterpret_cast<int4*>(ws);
    int32_t* optr = reinterpret_cast<int32_t*>(ell + nch * rpad);
    int32_t* ovf = optr + slots;
    int64_t* bsum = reinterpret_cast<int64_t*>(
        (reinterpret_cast<uintptr_t>(ovf + n * s) + 15) & ~uintptr_t(15));
    SKP_CUDA(cudaMemsetAsync(optr, 0, slots * sizeof(int32_t), st));
    const unsigned cb = (unsigned)std::min<int64_t>(cdiv(r, 128), 4096);
    ell_count_kernel<<<cb, 128, 0, st>>>(colptr, entries, r, J, optr);
    SKP_LAUNCHED(ell_count_kernel);
    const int64_t nb = cdiv(slots, kScanB * 8);
    scan_block_sums<<<(unsigned)nb, kScanB, 0, st>>>(optr, slots, bsum);
    SKP_LAUNCHED(scan_block_sums);
    scan_sums_serial<<<1, 32, 0, st>>>(bsum, nb, optr + slots - 1);
    SKP_LAUNCHED(scan_sums_serial);
    scan_apply<<<(unsigned)nb, kScanB, 0, st>>>(optr, slots - 1, bsum);
    SKP_LAUNCHED(scan_apply);
    const unsigned fb = (unsigned)std::min<int64_t>(cdiv(rpad, 128), 4096);
    ell_fill_kernel<<<fb, 128, 0, st>>>(colptr, entries, r, rpad, J, (int)nch, (int)sizeof(T),
                                        C::zero_off, optr, ell, ovf);
    SKP_LAUNCHED(ell_fill_kernel);

    const int P = (int)cdiv(r, C::SW);
    const int64_t blocks = cdiv(m, 32) * P;
    if (blocks > INT32_MAX) return SKP_ERR_UNSUPPORTED;
    SKP_CUDA(cudaFuncSetAttribute(sketch_rows_kernel<T>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::bytes));
    const T scale = T(1) / sqrt(T(s));
    sketch_rows_kernel<T><<<(unsigned)blocks, kRowsThreads, C::bytes, st>>>(
        A, lda, m, n, (int)nch, P, ell, ovf, optr, rpad, r, scale, out, ldo, fro2,
        reinterpret_cast<long long*>(nonfinite));
    SKP_LAUNCHED(sketch_rows_kernel);
    return SKP_OK;
}

template int sketch_right_rows<float>(const float*, int64_t, int64_t, int64_t, const int32_t*,
                                      const int32_t*, int32_t, int64_t, float*, int64_t, double*,
                                      int64_t*, void*, int64_t, cudaStream_t);
template int sketch_right_rows<double>(const double*, int64_t, int64_t, int64_t, const int32_t*,
                                       const int32_t*, int32_t, int64_t, double*, int64_t,
                                       double*, int64_t*, void*, int64_t, cudaStream_t);

int64_t sketch_rows_ws_bytes(int64_t n, int32_t s, int64_t r, int elem) {
    return elem == 8 ? rows_chunk_ws(n, s, r, RowsSmem<double>::J, RowsSmem<double>::SW)
                     : rows_chunk_ws(n, s, r, RowsSmem<float>::J, RowsSmem<float>::SW);
}

}  // namespace skp
