// K1 window_align (GenASM-DC + GenASM-TB + window loop) and K2/K3 CIGAR
// offset scan / compaction, hand-written for sm_100a. Design: DESIGN.md §3.
#include "window_align.cuh"

#include <cuda_runtime.h>

namespace sgk {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// Per limb-count tuning: R rows per register chunk, C traceback-code columns
// kept in shared memory (>= W-O for the supported O range),
// WARPS warps per block (warps are independent; blocks only share an SM).
template <int L> struct KCfg;
template <> struct KCfg<1> { static constexpr int R = 8, C = 32, WARPS = 4; };
template <> struct KCfg<2> { static constexpr int R = 8, C = 40, WARPS = 4; };
template <> struct KCfg<4> { static constexpr int R = 4, C = 32, WARPS = 2; };

template <int L> __host__ __device__ constexpr int txt_words() { return (32 * L / 8) * 32 * 2; }
template <int L> __host__ __device__ constexpr int pq_words() { return KCfg<L>::C * 2 * L * 32; }
template <int L> __host__ __device__ constexpr int pm_words() { return 5 * L * 32; }
template <int L> __host__ __device__ constexpr int warp_smem_words() {
    return txt_words<L>() + pq_words<L>() + pm_words<L>();
}

// ---------------------------------------------------------------- bit utils

// x holds bits only at multiples of S; returns them packed (bit k = bit kS).
template <int S> __device__ __forceinline__ uint32_t compress_stride(uint32_t x);
template <> __device__ __forceinline__ uint32_t compress_stride<1>(uint32_t x) { return x; }
template <> __device__ __forceinline__ uint32_t compress_stride<2>(uint32_t x) {
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    return (x | (x >> 8)) & 0x0000FFFFu;
}
template <> __device__ __forceinline__ uint32_t compress_stride<4>(uint32_t x) {
    x = (x | (x >> 3)) & 0x03030303u;
    x = (x | (x >> 6)) & 0x000F000Fu;
    return (x | (x >> 12)) & 0x000000FFu;
}
template <> __device__ __forceinline__ uint32_t compress_stride<8>(uint32_t x) {
    x = (x | (x >> 7)) & 0x00030003u;
    return (x | (x >> 14)) & 0x0000000Fu;
}
template <int S> __device__ __forceinline__ constexpr uint32_t stride_mask() {
    return S == 1 ? 0xFFFFFFFFu : S == 2 ? 0x55555555u : S == 4 ? 0x11111111u : 0x01010101u;
}

__device__ __forceinline__ uint32_t shr_sat(uint32_t x, int s) { return s >= 32 ? 0u : x >> s; }

// 4 two-bit fields (bits 0..7) -> 4 bytes; 4 bits -> 4 bytes of 0/1.
__device__ __forceinline__ uint32_t spread4(uint32_t a) {
    a &= 0xFFu;
    return (a | (a << 6) | (a << 12) | (a << 18)) & 0x03030303u;
}
__device__ __forceinline__ uint32_t spread4bits(uint32_t b) {
    b &= 0xFu;
    return (b | (b << 7) | (b << 14) | (b << 21)) & 0x01010101u;
}

// x*2 + b on the FMA pipe (IMAD): the DP shift of limb 0 into limb L-1.
__device__ __forceinline__ uint32_t dp_shift(uint32_t x, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 2, %2;" : "=r"(r) : "r"(x), "r"(b));
    return r;
}

// NW words of 2-bit codes starting at base `base` (base k at bits 2(k%16)).
template <int NW>
__device__ __forceinline__ void load_codes(const uint32_t* __restrict__ seq, int64_t base,
                                           uint32_t (&w)[NW]) {
    const uint32_t* src = seq + (base >> 4);
    const int s = static_cast<int>(base & 15) * 2;
    uint32_t prev = __ldg(src);
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        const uint32_t nx = __ldg(src + k + 1);
        w[k] = __funnelshift_r(prev, nx, s);
        prev = nx;
    }
}

// NW words of a 1-bit-per-base mask starting at base `base`.
template <int NW>
__device__ __forceinline__ void load_bits(const uint32_t* __restrict__ mask, int64_t base,
                                          uint32_t (&w)[NW]) {
    const uint32_t* src = mask + (base >> 5);
    const int s = static_cast<int>(base & 31);
    uint32_t prev = __ldg(src);
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        const uint32_t nx = __ldg(src + k + 1);
        w[k] = __funnelshift_r(prev, nx, s);
        prev = nx;
    }
}

// Bit plane b of the 2-bit codes of the bases j = rho + kL (bit k of result).
template <int L>
__device__ __forceinline__ uint32_t gather_codes(const uint32_t (&pw)[2 * L], int rho, int b) {
    constexpr int S = 2 * L, PER = 16 / L;
    uint32_t g = 0;
#pragma unroll
    for (int k = 0; k < 2 * L; ++k)
        g |= compress_stride<S>((pw[k] >> (2 * rho + b)) & stride_mask<S>()) << (k * PER);
    return g;
}

// Bits j = rho + kL of a 1-bit-per-base mask (bit k of result).
template <int L>
__device__ __forceinline__ uint32_t gather_bits(const uint32_t (&nw)[L], int rho) {
    constexpr int PER = 32 / L;
    uint32_t g = 0;
#pragma unroll
    for (int k = 0; k < L; ++k)
        g |= compress_stride<L>((nw[k] >> rho) & stride_mask<L>()) << (k * PER);
    return g;
}

// Limb r of a right-aligned vector built from per-class gathers: base j of
// the chunk sits at q = j + off, limb q % L, machine bit 31 - q / L.
template <int L>
__device__ __forceinline__ uint32_t limbify(uint32_t g_rho, int r, int off, int rho) {
    const int s = (off + rho - r) / L;  // >= 0
    return shr_sat(__brev(g_rho), s);
}

template <int L> __device__ __forceinline__ int class_of(int r, int off) {
    return ((r - off) % L + L) % L;
}

// R[n][d] for the init column (proj/src/dp.cpp:146,179): ones << min(d, m),
// i.e. the lowest d logical positions cleared.
template <int L> __device__ __forceinline__ uint32_t init_limb(int d, int l) {
    if (d < 0) return ~0u;
    const int z = (d + l) / L;
    return z >= 32 ? 0u : (~0u << z);
}

__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// ---------------------------------------------------------------- skewed DC sweep
//
// One chunk (rows d0..d0+R-1) of GenASM-DC over all columns of a window as a
// skewed wavefront: at step s row r works on column col0(s) + r, where
// col0(s) = S0 - s is row 0's column. The R cells of a step are independent
// (each needs only the previous step's values), which gives the warp R-way
// instruction-level parallelism instead of an R-long dependency chain.
// Columns >= n_w are "virtual": pattern mask all ones and boundary bits 0,
// which reproduce the init column R[n][d] exactly, so the fill of the
// wavefront needs no special code. The pattern masks and the traceback event
// accumulators of the R columns in flight live in rings indexed by the step
// at which row 0 entered the column; unrolling the step loop by R makes every
// ring index static (no register moves).
template <int L, int R>
struct Sweep {
    uint32_t v[R][L];       // latest value of row r (R[col_r][d0 + r])
    uint32_t dg[R][L];      // diag input of row r at its next step
    uint32_t ic[R];         // S(col_r - 1, d) = shifted limb of I(col_r, d)
    uint32_t pmq[R][L];     // pattern mask ring
    uint32_t acc[R][2][L];  // X / Y event ring
};

// Step U (static) of a group. MODE 0: fast, no capture; 1: fast with capture;
// 2: slow (explicit boundary bits) with capture. `g` = n_w - S0 - d0 + s; the
// boundary bits of row r are [g >= 2r] (plus d == 0 for row 0) and [g >= 2r+2]
// (dp.cpp:187-195 with c = n_w - col: [c > d-1], [c-1 > d]).
template <int L, int R, int U, int MODE>
__device__ __forceinline__ void sweep_step(Sweep<L, R>& S, const uint32_t (&north0)[L],
                                           const uint32_t (&pm0)[L], int g, bool z0) {
#pragma unroll
    for (int l = 0; l < L; ++l) S.pmq[U][l] = pm0[l];
    uint32_t t[R + 1];
    if (MODE == 2) {
#pragma unroll
        for (int k = 0; k <= R; ++k) t[k] = static_cast<uint32_t>(g >= 2 * k);
        t[0] |= static_cast<uint32_t>(z0);
    }
#pragma unroll
    for (int r = R - 1; r >= 0; --r) {
        constexpr int dummy = 0;
        (void)dummy;
        const int slot = (U - r) & (R - 1);
        uint32_t north[L], east[L], diag[L], pm[L];
#pragma unroll
        for (int l = 0; l < L; ++l) {
            north[l] = r == 0 ? north0[l] : S.v[r == 0 ? 0 : r - 1][l];
            east[l] = S.v[r][l];
            diag[l] = S.dg[r][l];
            pm[l] = S.pmq[slot][l];
        }
        const uint32_t bI = MODE == 2 ? t[r] : 1u;
        const uint32_t bM = MODE == 2 ? t[r + 1] : 1u;
        uint32_t I[L], M[L], Sv[L], Rv[L];
#pragma unroll
        for (int l = 0; l + 1 < L; ++l) {
            I[l] = north[l + 1];
            M[l] = east[l + 1];
            Sv[l] = diag[l + 1];
        }
        I[L - 1] = dp_shift(north[0], bI);
        M[L - 1] = dp_shift(east[0], bM);
        Sv[L - 1] = S.ic[r];
#pragma unroll
        for (int l = 0; l < L; ++l) Rv[l] = I[l] & diag[l] & Sv[l] & (M[l] | pm[l]);
        if (MODE != 0) {
#pragma unroll
            for (int l = 0; l < L; ++l) {
                const uint32_t x = Rv[l] & ~M[l], y = Rv[l] & ~east[l];
                if (r == 0) {
                    S.acc[slot][0][l] = x;
                    S.acc[slot][1][l] = y;
                } else {
                    S.acc[slot][0][l] |= x;
                    S.acc[slot][1][l] |= y;
                }
            }
        }
        S.ic[r] = I[L - 1];
#pragma unroll
        for (int l = 0; l < L; ++l) {
            if (r + 1 < R) S.dg[r + 1 < R ? r + 1 : 0][l] = east[l];
            S.v[r][l] = Rv[l];
        }
    }
#pragma unroll
    for (int l = 0; l < L; ++l) S.dg[0][l] = north0[l];
}

// Drain step K (1..R-1, static): row 0's column is -K; rows r >= K finish
// columns r-K. Boundary bits explicit (MODE 2 rule).
template <int L, int R, int K>
__device__ __forceinline__ void drain_step(Sweep<L, R>& S, int g) {
    uint32_t t[R + 1];
#pragma unroll
    for (int k = 0; k <= R; ++k) t[k] = static_cast<uint32_t>(g >= 2 * k);
#pragma unroll
    for (int r = R - 1; r >= K; --r) {
        const int slot = (R - 1 + K - r) & (R - 1);
        uint32_t north[L], east[L], diag[L], pm[L];
#pragma unroll
        for (int l = 0; l < L; ++l) {
            north[l] = S.v[r - 1][l];
            east[l] = S.v[r][l];
            diag[l] = S.dg[r][l];
            pm[l] = S.pmq[slot][l];
        }
        uint32_t I[L], M[L], Sv[L], Rv[L];
#pragma unroll
        for (int l = 0; l + 1 < L; ++l) {
            I[l] = north[l + 1];
            M[l] = east[l + 1];
            Sv[l] = diag[l + 1];
        }
        I[L - 1] = dp_shift(north[0], t[r]);
        M[L - 1] = dp_shift(east[0], t[r + 1]);
        Sv[L - 1] = S.ic[r];
#pragma unroll
        for (int l = 0; l < L; ++l) Rv[l] = I[l] & diag[l] & Sv[l] & (M[l] | pm[l]);
#pragma unroll
        for (int l = 0; l < L; ++l) {
            S.acc[slot][0][l] |= Rv[l] & ~M[l];
            S.acc[slot][1][l] |= Rv[l] & ~east[l];
        }
        S.ic[r] = I[L - 1];
#pragma unroll
        for (int l = 0; l < L; ++l) {
            if (r + 1 < R) S.dg[r + 1 < R ? r + 1 : 0][l] = east[l];
            S.v[r][l] = Rv[l];
        }
    }
}

// Side effects of the column row R-1 just finished (static ring SLOT): park
// its value for the next chunk and fold the column's events into the 2-bit
// traceback codes P = X | ~PM, Q = PM & (X | Y)  (M=(1,0) S=(1,1) D=(0,1) I=(0,0)).
template <int L, int R, int C, int SLOT, bool CAP>
__device__ __forceinline__ void finish_col(const Sweep<L, R>& S, int colf, int n_w, int d0,
                                           uint32_t* __restrict__ pq, uint32_t* __restrict__ bnd,
                                           int lane) {
    if (colf >= 0 && colf < n_w) {
#pragma unroll
        for (int l = 0; l < L; ++l) bnd[(colf * 32 + lane) * L + l] = S.v[R - 1][l];
        if (CAP && colf < C) {
#pragma unroll
            for (int l = 0; l < L; ++l) {
                uint32_t* pp = pq + ((colf * 2 + 0) * L + l) * 32 + lane;
                uint32_t* qp = pq + ((colf * 2 + 1) * L + l) * 32 + lane;
                const uint32_t pm = S.pmq[SLOT][l];
                const uint32_t x = S.acc[SLOT][0][l], y = S.acc[SLOT][1][l];
                const uint32_t pold = d0 > 0 ? *pp : ~pm;
                const uint32_t qold = d0 > 0 ? *qp : 0u;
                *pp = pold | x;
                *qp = qold | (pm & (x | y));
            }
        }
    }
}

// Bit j = 0 of row r's value at column 0 (the d_opt test, dp.cpp:222).
template <int L, int R>
__device__ __forceinline__ uint32_t top_bit(const Sweep<L, R>& S, int r, int r0, int p0) {
    uint32_t v = S.v[r][0];
#pragma unroll
    for (int l = 1; l < L; ++l) v = r0 == l ? S.v[r][l] : v;
    return (v >> (31 - p0)) & 1u;
}

template <int L, int R, int C, int MODE>
__device__ __forceinline__ void sweep_group(Sweep<L, R>& S, const uint32_t (&nb)[R][L],
                                            uint64_t codes8, int col_top,
                                            const uint32_t* __restrict__ pmv, int g0, bool z0,
                                            int n_w, int d0, uint32_t* __restrict__ pq,
                                            uint32_t* __restrict__ bnd, int lane) {
#define SG_STEP(U)                                                                          \
    if ((U) < R) {                                                                          \
        const int col0 = col_top - (U);                                                     \
        const int code = static_cast<int>((codes8 >> (8 * (col0 & 7))) & 0xFFu);            \
        uint32_t pm0[L];                                                                    \
        _Pragma("unroll") for (int l = 0; l < L; ++l) pm0[l] = pmv[(code * 32 + lane) * L + l]; \
        sweep_step<L, R, ((U) < R ? (U) : 0), MODE>(S, nb[(U) < R ? (U) : 0], pm0, g0 + (U), z0); \
        finish_col<L, R, C, (((U) + 1) & (R - 1)), MODE != 0>(S, col0 + R - 1, n_w, d0, pq, bnd, \
                                                            lane);                           \
    }
    SG_STEP(0) SG_STEP(1) SG_STEP(2) SG_STEP(3) SG_STEP(4) SG_STEP(5) SG_STEP(6) SG_STEP(7)
#undef SG_STEP
}

template <int L, int R, int C, int K>
__device__ __forceinline__ void drain_one(Sweep<L, R>& S, int g, int n_w, int d0, uint32_t* pq,
                                          uint32_t* bnd, int lane, int r0, int p0, int& fr) {
    if (K < R) {
        drain_step<L, R, (K < R ? K : 1)>(S, g);
        finish_col<L, R, C, (K & (R - 1)), true>(S, R - 1 - K, n_w, d0, pq, bnd, lane);
        if (fr < 0 && !top_bit<L, R>(S, K < R ? K : 0, r0, p0)) fr = K;
    }
}

// One chunk of rows d0..d0+R-1 over columns n_w-1..0 (n_w = 0: inactive lane).
// Returns the first row r of the chunk with bit j=0 of R[0][d0+r] clear, or -1.
template <int L, int R, int C>
__device__ __forceinline__ int dc_chunk(int n_w, int m_w, int d0, int n_max,
                                        const uint32_t* __restrict__ pmv,
                                        const uint64_t* __restrict__ txt, uint32_t* __restrict__ pq,
                                        uint32_t* __restrict__ bnd, int lane) {
    constexpr int WB = 32 * L;
    static_assert((R & (R - 1)) == 0 && R <= 8 && WB % R == 0, "R must be a power of two <= 8");
    Sweep<L, R> S;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int d = d0 + r;
#pragma unroll
        for (int l = 0; l < L; ++l) {
            S.v[r][l] = init_limb<L>(d, l);
            S.dg[r][l] = init_limb<L>(d - 1, l);
            S.pmq[r][l] = ~0u;
            S.acc[r][0][l] = S.acc[r][1][l] = 0u;
        }
        // I(n, d) = shl1(R[n][d-1], [d == 0]) with R[n][-1] = ones
        S.ic[r] = d == 0 ? ~0u : (init_limb<L>(d - 1, 0) << 1);
    }
    const int tsteps = ((n_max + R - 1) / R) * R;
    const int S0 = tsteps - 1;
    const bool z0 = d0 == 0;
    uint32_t init_north[L];
#pragma unroll
    for (int l = 0; l < L; ++l) init_north[l] = init_limb<L>(d0 - 1, l);
    // row-0 north inputs (the parked row d0-1), prefetched one group ahead
    uint32_t nb[R][L], nbn[R][L];
    auto fetch_nb = [&](uint32_t (&dst)[R][L], int col_top) {
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int col = col_top - u;
            const bool real = col >= 0 && col < n_w && d0 > 0;
#pragma unroll
            for (int l = 0; l < L; ++l)
                dst[u][l] = real ? bnd[(col * 32 + lane) * L + l] : init_north[l];
        }
    };
    fetch_nb(nb, S0);
    for (int sg = 0; sg < tsteps; sg += R) {
        const int col_top = S0 - sg;
        if (sg + R < tsteps) fetch_nb(nbn, col_top - R);
        const uint64_t codes8 = txt[(col_top >> 3) * 32 + lane];
        const int g0 = n_w - S0 - d0 + sg;
        const bool slow = __any_sync(kFull, n_w > 0 && g0 < 2 * R);
        if (slow)
            sweep_group<L, R, C, 2>(S, nb, codes8, col_top, pmv, g0, z0, n_w, d0, pq, bnd, lane);
        else if (col_top - R + 1 < C)
            sweep_group<L, R, C, 1>(S, nb, codes8, col_top, pmv, g0, z0, n_w, d0, pq, bnd, lane);
        else
            sweep_group<L, R, C, 0>(S, nb, codes8, col_top, pmv, g0, z0, n_w, d0, pq, bnd, lane);
#pragma unroll
        for (int u = 0; u < R; ++u)
#pragma unroll
            for (int l = 0; l < L; ++l) nb[u][l] = nbn[u][l];
    }
    const int off = WB - m_w;
    const int r0 = off % L, p0 = off / L;
    int fr = top_bit<L, R>(S, 0, r0, p0) ? -1 : 0;
    const int gd = n_w - S0 - d0 + tsteps;  // g at drain step 1 minus 1
    drain_one<L, R, C, 1>(S, gd + 0, n_w, d0, pq, bnd, lane, r0, p0, fr);
    drain_one<L, R, C, 2>(S, gd + 1, n_w, d0, pq, bnd, lane, r0, p0, fr);
    drain_one<L, R, C, 3>(S, gd + 2, n_w, d0, pq, bnd, lane, r0, p0, fr);
    drain_one<L, R, C, 4>(S, gd + 3, n_w, d0, pq, bnd, lane, r0, p0, fr);
    drain_one<L, R, C, 5>(S, gd + 4, n_w, d0, pq, bnd, lane, r0, p0, fr);
    drain_one<L, R, C, 6>(S, gd + 5, n_w, d0, pq, bnd, lane, r0, p0, fr);
    drain_one<L, R, C, 7>(S, gd + 6, n_w, d0, pq, bnd, lane, r0, p0, fr);
    return fr;
}

// ------------------------------------------------------------------ K1

template <int L>
__global__ void __launch_bounds__(32 * KCfg<L>::WARPS)
    k1_window_align(const AlignParams P) {
    constexpr int R = KCfg<L>::R, C = KCfg<L>::C, WB = 32 * L;
    extern __shared__ uint32_t smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    uint64_t* const txt = reinterpret_cast<uint64_t*>(smem + wib * warp_smem_words<L>());
    uint32_t* const pq = smem + wib * warp_smem_words<L>() + txt_words<L>();  // [C][2][L][32]
    uint32_t* const pmv = pq + pq_words<L>();                                 // [5][32][L]
    const long long gwarp = static_cast<long long>(blockIdx.x) * KCfg<L>::WARPS + wib;
    uint32_t* const bnd = P.bnd + gwarp * (WB + 1) * 32 * L;  // [WB+1][32][L]

#pragma unroll
    for (int l = 0; l < L; ++l) pmv[(4 * 32 + lane) * L + l] = ~0u;  // non-ACGT text

    const int W = P.W;
    const int step_limit = W - P.O;

    // ---- lane state ----
    int pair = -1;
    int n_tot = 0, m_tot = 0;
    int64_t tbase = 0, pbase = 0;
    bool hasn = false;
    int toff = 0, poff = 0, n_w = 0, m_w = 0, limit = 0;
    bool first_seg = true;
    int d0 = 0, found_d = -1, expect_d = -1;
    int dist = 0, nwin = 0, status = 0;
    long long window_cap = 0;
    // output
    uint32_t* outw = nullptr;
    int out_bytes = 0, cur_op = -1, acc_n = 0;
    long long cur_len = 0;
    uint32_t acc = 0;
    // counters (InstrumentationCounters, proj/include/scrooge/dp.hpp:46-66)
    unsigned long long c_stored = 0, c_writes = 0, c_reads = 0, c_rows = 0, c_cells = 0,
                       c_bequiv = 0;

    auto put_byte = [&](uint32_t b) {
        acc |= b << (8 * acc_n);
        ++out_bytes;
        if (++acc_n == 4) {
            *outw++ = acc;
            acc = 0;
            acc_n = 0;
        }
    };
    auto flush_run = [&]() {
        if (cur_op < 0) return;
        long long len = cur_len;
        const uint32_t hi = static_cast<uint32_t>(cur_op) << 6;
        while (len > 64) {
            put_byte(hi | 63u);
            len -= 64;
        }
        put_byte(hi | static_cast<uint32_t>(len - 1));
        cur_op = -1;
        cur_len = 0;
    };
    auto emit = [&](int op, long long len) {  // cigar_append, proj/src/cigar.cpp:9-16
        if (op == cur_op) {
            cur_len += len;
        } else {
            flush_run();
            cur_op = op;
            cur_len = len;
        }
    };

    // Pattern masks and text codes of the current segment.
    auto load_segment = [&]() {
        const int off = WB - m_w;
        uint32_t pw[2 * L];
        load_codes<2 * L>(P.seq, pbase + poff, pw);
        uint32_t pn[L];
#pragma unroll
        for (int l = 0; l < L; ++l) pn[l] = 0;
        if (hasn) load_bits<L>(P.nmask, pbase + poff, pn);
#pragma unroll
        for (int r = 0; r < L; ++r) {
            const int rho = class_of<L>(r, off);
            const uint32_t lo = limbify<L>(gather_codes<L>(pw, rho, 0), r, off, rho);
            const uint32_t hi = limbify<L>(gather_codes<L>(pw, rho, 1), r, off, rho);
            const uint32_t nn = hasn ? limbify<L>(gather_bits<L>(pn, rho), r, off, rho) : 0u;
            // PM[c] bit = 0 iff pattern base == c (proj/src/dp.cpp:8-21); N matches nothing
            pmv[(0 * 32 + lane) * L + r] = lo | hi | nn;
            pmv[(1 * 32 + lane) * L + r] = ~lo | hi | nn;
            pmv[(2 * 32 + lane) * L + r] = lo | ~hi | nn;
            pmv[(3 * 32 + lane) * L + r] = ~lo | ~hi | nn;
        }
        uint32_t tw[2 * L], tn[L];
        load_codes<2 * L>(P.seq, tbase + toff, tw);
#pragma unroll
        for (int l = 0; l < L; ++l) tn[l] = 0;
        if (hasn) load_bits<L>(P.nmask, tbase + toff, tn);
        // text codes as bytes, 8 columns per u64; non-ACGT and columns >= n_w -> 4
#pragma unroll
        for (int b = 0; b < WB / 8; ++b) {
            const uint32_t x = (tw[b >> 1] >> (16 * (b & 1))) & 0xFFFFu;
            uint64_t c = static_cast<uint64_t>(spread4(x)) |
                         (static_cast<uint64_t>(spread4(x >> 8)) << 32);
            const uint32_t nb8 = (tn[b >> 2] >> (8 * (b & 3))) & 0xFFu;
            uint64_t m = (static_cast<uint64_t>(spread4bits(nb8)) |
                          (static_cast<uint64_t>(spread4bits(nb8 >> 4)) << 32)) * 0xFFull;
            const int valid = n_w - 8 * b;
            if (valid < 8) m |= valid <= 0 ? ~0ull : (~0ull << (8 * valid));
            c = (c & ~m) | (0x0404040404040404ull & m);
            txt[b * 32 + lane] = c;
        }
    };

    // Sets up the next logical window of the current pair (aligner.cpp:44-64).
    // Returns false when the pair is complete (residues appended).
    auto next_window = [&]() -> bool {
        const int n_rem = n_tot - toff, m_rem = m_tot - poff;
        if (n_rem == 0 && m_rem == 0) return false;
        if (n_rem == 0) {
            emit(2, m_rem);
            dist += m_rem;
            return false;
        }
        if (m_rem == 0) {
            emit(3, n_rem);
            dist += n_rem;
            return false;
        }
        const bool fin = n_rem <= W && m_rem <= W;
        n_w = min(W, n_rem);
        m_w = min(W, m_rem);
        limit = fin ? -1 : step_limit;
        first_seg = true;
        d0 = 0;
        found_d = -1;
        expect_d = -1;
        load_segment();
        return true;
    };

    auto finish_pair = [&]() {
        flush_run();
        if (acc_n) *outw = acc;
        P.distance[pair] = dist;
        P.windows[pair] = nwin;
        P.status[pair] = status;
        P.out_bytes[pair] = out_bytes;
        if (P.counters) {
            uint64_t* c = P.counters + 7ll * pair;
            c[0] = c_stored;
            c[1] = c_writes;
            c[2] = c_reads;
            c[3] = c_rows;
            c[4] = c_cells;
            c[5] = static_cast<unsigned long long>(nwin) * static_cast<unsigned>(W + 1);
            c[6] = c_bequiv;
        }
    };

    auto start_pair = [&](int q) {
        pair = q < P.n_pairs ? (P.order ? P.order[q] : q) : -1;
        if (pair < 0) return;
        n_tot = P.text_len[pair];
        m_tot = P.pat_len[pair];
        tbase = P.text_off[pair];
        pbase = P.pat_off[pair];
        hasn = P.has_n ? P.has_n[pair] != 0 : false;
        toff = poff = 0;
        dist = nwin = status = 0;
        window_cap = 4ll * ((static_cast<long long>(n_tot) + m_tot) / step_limit + 2);
        outw = P.scratch + (P.bound_off[pair] >> 2);
        out_bytes = 0;
        cur_op = -1;
        cur_len = 0;
        acc = 0;
        acc_n = 0;
        c_stored = c_writes = c_reads = c_rows = c_cells = c_bequiv = 0;
    };

    // Claim the next pair(s) for the calling (possibly divergent) lanes.
    auto fetch = [&]() {
        const unsigned active = __activemask();
        const int leader = __ffs(active) - 1;
        unsigned base = 0;
        if (lane == leader) base = atomicAdd(P.next_pair, static_cast<unsigned>(__popc(active)));
        base = __shfl_sync(active, base, leader);
        const int q = static_cast<int>(base + __popc(active & ((1u << lane) - 1u)));
        start_pair(q);
    };

    fetch();
    while (pair >= 0 && !next_window()) {  // cannot happen for valid pairs (n, m >= 1)
        finish_pair();
        fetch();
    }

    for (;;) {
        const bool in_dc = pair >= 0;
        if (!__any_sync(kFull, in_dc)) break;

        // ------------------------------------------------ DC: one chunk
        const int n_max = warp_max(in_dc ? n_w : 0);
        const int fr = dc_chunk<L, R, C>(in_dc ? n_w : 0, m_w, d0, n_max, pmv, txt, pq, bnd, lane);

        // ------------------------------------------------ d_opt detection
        bool solved = false;
        if (in_dc) {
            if (found_d < 0 && fr >= 0) found_d = d0 + fr;
            const bool seg_et = P.et || !first_seg;
            solved = seg_et ? found_d >= 0 : (d0 + R > W);
            if (!solved) d0 += R;
        }

        // ------------------------------------------------ TB + advance
        if (in_dc && solved) {
            if (found_d < 0) status = kStInternal | kDetNoStep;  // aligner.cpp:69-70
            if (first_seg) {
                // reference counters for this logical window (dp.cpp:23-37,58-75,225-228)
                const int rows_ref = P.et ? found_d + 1 : W + 1;
                int pol = P.policy;
                if (limit < 0 && pol == 2) pol = 1;  // final window: DENT -> SENE
                int keep_cols = n_w + 1, keep_bits = m_w;
                if (pol == 2) {
                    keep_cols = min(n_w, step_limit) + 1;
                    keep_bits = min(m_w, step_limit + 1);
                }
                const unsigned long long slots = pol == 0 ? 3ull : 1ull;
                c_stored += static_cast<unsigned long long>(rows_ref) * keep_cols * keep_bits * slots;
                c_writes += static_cast<unsigned long long>(rows_ref) * keep_cols * slots;
                c_rows += rows_ref;
                c_cells += static_cast<unsigned long long>(rows_ref) * n_w;
                c_bequiv += 3ull * (n_w + 1) * static_cast<unsigned long long>(W + 1) * m_w;
            } else if (found_d != expect_d) {
                status = kStInternal | kDetSegment;
            }
            // GenASM-TB (traceback.cpp:56-113) over the 2-bit codes
            const int off = WB - m_w;
            int i = 0, j = 0, d = found_d < 0 ? 0 : found_d, steps = 0;
            bool cont = false;
            for (;;) {
                if (limit >= 0 && steps == limit) break;
                if (i == n_w && j == m_w) break;
                int op;
                if (i == n_w) {
                    if (d != m_w - j) status = kStInternal | kDetBudgetI;
                    op = 2;
                } else if (j == m_w) {
                    if (d != n_w - i) status = kStInternal | kDetBudgetD;
                    op = 3;
                } else if (i >= C) {
                    cont = true;
                    break;
                } else {
                    c_reads += d == 0 ? 1 : 3;
                    const int q = j + off;
                    const int r = q % L, p = q / L;
                    const uint32_t pw = pq[((i * 2 + 0) * L + r) * 32 + lane];
                    const uint32_t qw = pq[((i * 2 + 1) * L + r) * 32 + lane];
                    const int pb = static_cast<int>((pw >> (31 - p)) & 1u);
                    const int qb = static_cast<int>((qw >> (31 - p)) & 1u);
                    op = qb | ((pb ^ 1) << 1);
                    if (op != 0 && d == 0) {
                        status = kStInternal | kDetNoStep;
                        op = 0;
                    }
                }
                i += op != 2;
                j += op != 3;
                d -= op != 0;
                ++steps;
                if (op != 0) ++dist;
                emit(op, 1);
            }
            if (cont && status == 0) {
                // the window continues on the suffix t[i:n_w) x p[j:m_w)
                toff += i;
                poff += j;
                n_w -= i;
                m_w -= j;
                if (limit >= 0) limit -= steps;
                first_seg = false;
                d0 = 0;
                found_d = -1;
                expect_d = d;
                load_segment();
            } else {
                if (!cont && limit < 0 && d != 0) status = kStInternal | kDetLeftover;
                toff += i;
                poff += j;
                ++nwin;
                if (nwin > window_cap) status = kStInternal | kDetWatchdog;
                bool more = status == 0 && next_window();
                while (!more) {
                    finish_pair();
                    fetch();
                    if (pair < 0) break;
                    more = next_window();
                }
            }
        }
    }
}

template <int L> size_t smem_bytes() {
    return static_cast<size_t>(warp_smem_words<L>()) * 4 * KCfg<L>::WARPS;
}

template <int L> int launch_L(const AlignParams& p, int grid, void* stream) {
    const size_t smem = smem_bytes<L>();
    cudaError_t e = cudaFuncSetAttribute(k1_window_align<L>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
    k1_window_align<L><<<grid, 32 * KCfg<L>::WARPS, smem, static_cast<cudaStream_t>(stream)>>>(p);
    return static_cast<int>(cudaGetLastError());
}

// ------------------------------------------------------------------ K2 / K3

constexpr int kScanBlock = 1024;

__device__ __forceinline__ long long warp_incl_scan(long long v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Block-level exclusive scan of the run byte counts; block totals to `sums`.
__global__ void __launch_bounds__(kScanBlock)
    k2_scan_blocks(const int32_t* __restrict__ bytes, int64_t* __restrict__ out, int32_t n,
                   long long* __restrict__ sums) {
    __shared__ long long warp_tot[kScanBlock / 32];
    const int idx = blockIdx.x * kScanBlock + threadIdx.x;
    const long long v = idx < n ? bytes[idx] : 0;
    const long long inc = warp_incl_scan(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    if (w == 0) {
        const long long t = warp_incl_scan(lane < kScanBlock / 32 ? warp_tot[lane] : 0);
        if (lane < kScanBlock / 32) warp_tot[lane] = t;
    }
    __syncthreads();
    const long long base = w > 0 ? warp_tot[w - 1] : 0;
    if (idx < n) out[idx] = base + inc - v;
    if (threadIdx.x == kScanBlock - 1) sums[blockIdx.x] = base + inc;
}

// Single-block exclusive scan of the block totals (loops for any count).
__global__ void __launch_bounds__(kScanBlock) k2_scan_sums(long long* __restrict__ sums, int nb,
                                                          int64_t* __restrict__ total) {
    __shared__ long long warp_tot[kScanBlock / 32];
    __shared__ long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += kScanBlock) {
        const int idx = base + threadIdx.x;
        const long long v = idx < nb ? sums[idx] : 0;
        const long long inc = warp_incl_scan(v);
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        if (lane == 31) warp_tot[w] = inc;
        __syncthreads();
        if (w == 0) {
            const long long t = warp_incl_scan(lane < kScanBlock / 32 ? warp_tot[lane] : 0);
            if (lane < kScanBlock / 32) warp_tot[lane] = t;
        }
        __syncthreads();
        const long long wbase = w > 0 ? warp_tot[w - 1] : 0;
        if (idx < nb) sums[idx] = carry + wbase + inc - v;
        __syncthreads();
        if (threadIdx.x == kScanBlock - 1) carry += wbase + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void k2_add(int64_t* __restrict__ out, int32_t n, const long long* __restrict__ sums) {
    const int idx = blockIdx.x * kScanBlock + threadIdx.x;
    if (idx < n) out[idx] += sums[blockIdx.x];
}

// One warp per pair copies its run bytes to their dense (unaligned) position:
// each lane assembles whole destination words from the source stream.
__global__ void k3_compact(const uint32_t* __restrict__ scratch, const int64_t* __restrict__ bound,
                           const int64_t* __restrict__ dense_off, const int32_t* __restrict__ bytes,
                           uint8_t* __restrict__ dense, int32_t n) {
    const int lane = threadIdx.x & 31;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long p = warp; p < n; p += nwarps) {
        const int nb = bytes[p];
        const uint8_t* src = reinterpret_cast<const uint8_t*>(scratch) + bound[p];
        uint8_t* dst = dense + dense_off[p];
        for (int k = lane; k < nb; k += 32) dst[k] = src[k];
    }
}

}  // namespace

int launch_window_align(int L, const AlignParams& p, int grid, int warps_per_block, void* stream) {
    (void)warps_per_block;
    switch (L) {
        case 1: return launch_L<1>(p, grid, stream);
        case 2: return launch_L<2>(p, grid, stream);
        case 4: return launch_L<4>(p, grid, stream);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

size_t bnd_scratch_bytes(int L, long long total_warps) {
    return static_cast<size_t>(total_warps) * static_cast<size_t>(32 * L + 1) * 32 * L * 4;
}

int k1_warps_per_block(int L) {
    return L == 1 ? KCfg<1>::WARPS : L == 2 ? KCfg<2>::WARPS : KCfg<4>::WARPS;
}

size_t k1_smem_bytes(int L) {
    return L == 1 ? smem_bytes<1>() : L == 2 ? smem_bytes<2>() : smem_bytes<4>();
}

int k1_max_blocks_per_sm(int L) {
    int blocks = 0;
    cudaError_t e;
    if (L == 1) {
        cudaFuncSetAttribute(k1_window_align<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_bytes<1>()));
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k1_window_align<1>,
                                                          32 * KCfg<1>::WARPS, smem_bytes<1>());
    } else if (L == 2) {
        cudaFuncSetAttribute(k1_window_align<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_bytes<2>()));
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k1_window_align<2>,
                                                          32 * KCfg<2>::WARPS, smem_bytes<2>());
    } else {
        cudaFuncSetAttribute(k1_window_align<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_bytes<4>()));
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k1_window_align<4>,
                                                          32 * KCfg<4>::WARPS, smem_bytes<4>());
    }
    return e == cudaSuccess ? blocks : 0;
}

size_t cigar_offsets_temp_bytes(int32_t n) {
    const int nb = (n + kScanBlock - 1) / kScanBlock;
    return static_cast<size_t>(nb + 1) * sizeof(long long);
}

int launch_cigar_offsets(const int32_t* out_bytes, int64_t* dense_off, int32_t n, void* temp,
                         size_t temp_bytes, void* stream) {
    const int nb = (n + kScanBlock - 1) / kScanBlock;
    if (temp_bytes < cigar_offsets_temp_bytes(n)) return static_cast<int>(cudaErrorInvalidValue);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    long long* sums = static_cast<long long*>(temp);
    // dense_off has n + 1 entries; the total lands in dense_off[n]
    if (nb > 0) {
        k2_scan_blocks<<<nb, kScanBlock, 0, s>>>(out_bytes, dense_off, n, sums);
        k2_scan_sums<<<1, kScanBlock, 0, s>>>(sums, nb, dense_off + n);
        k2_add<<<nb, kScanBlock, 0, s>>>(dense_off, n, sums);
    } else {
        cudaMemsetAsync(dense_off, 0, sizeof(int64_t), s);
    }
    return static_cast<int>(cudaGetLastError());
}

int launch_cigar_compact(const uint32_t* scratch, const int64_t* bound_off, const int64_t* dense_off,
                         const int32_t* out_bytes, uint8_t* dense, int32_t n, void* stream) {
    if (n <= 0) return 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int threads = 256;
    long long blocks = (static_cast<long long>(n) * 32 + threads - 1) / threads;
    if (blocks > 8ll * sms) blocks = 8ll * sms;
    k3_compact<<<static_cast<int>(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(
        scratch, bound_off, dense_off, out_bytes, dense, n);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace sgk
