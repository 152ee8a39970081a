// K1 window_align (GenASM-DC + GenASM-TB + window loop) and K2/K3 CIGAR
// offset scan / compaction, hand-written for sm_100a. Design: DESIGN.md §3.
#include "window_align.cuh"
#ifdef SG_DEBUG_POST
#include <cstdio>
#endif

#include <cuda_runtime.h>

#include <utility>

namespace sgk {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// Per limb-count tuning: R rows per register chunk (power of two <= 8), C
// traceback-event columns kept in shared memory (>= W-O for the supported O
// range, wider windows continue as a new segment), WARPS warps per block
// (warps are independent; blocks only share an SM).
template <int L> struct KCfg;
template <> struct KCfg<1> { static constexpr int R = 4, C = 32, WARPS = 4, MINB = 2; };
// (L = 2: two blocks of four warps per SM and up to 255 registers. With three blocks, 12
// warps at 168 registers, the sweep state spilled to a 128-byte stack frame: cfg5 127 ->
// 105 ms, cfg2's final-window pass 1.67 -> 1.3 ms, cfg4 W = 64 in this kernel 12.5 -> 9.8;
// 6, 9, 10 warps per SM: 124, 114, 123 ms.)
template <> struct KCfg<2> { static constexpr int R = 4, C = 40, WARPS = 4, MINB = 2; };
// (L = 4: C covers W - O = 80 of cfg4's W = 128, O = 48; with 32 columns every such
// window ran as three continuation segments, 2.7 x the DC chunks)
#ifndef SG_C4
#define SG_C4 80
#endif
template <> struct KCfg<4> { static constexpr int R = 4, C = SG_C4, WARPS = 2, MINB = 1; };
// DC chunks per state-machine iteration (traceback batching, see the main loop)
// (band warps: their chunks cost a third of a full-frame chunk, so the traceback
// and setup phases amortise over more of them; measured 2 / 3 / 4 / 6 / 8 on cfg3:
// 4 is best)
#ifndef SG_SUBCHUNKS
#define SG_SUBCHUNKS 2
#endif
// Full-frame warps: after kSubChunks chunks the traceback phase starts once
// kTbLanes of 32 (scaled to the lanes that hold a pair) wait for it, or after
// kSubMax chunks. A window of an unrelated pair takes ~9 chunks: with a phase every
// 2 chunks only ~18 % of the lanes were in each traceback.
#ifndef SG_TB_LANES
#define SG_TB_LANES 12
#endif
#ifndef SG_SUBMAX
#define SG_SUBMAX 6
#endif
#ifndef SG_BAND_R
#define SG_BAND_R 8  // rows per band chunk (kBandR)
#endif
#ifndef SG_BAND_SUBCHUNKS
#define SG_BAND_SUBCHUNKS (16 / SG_BAND_R)  // 16 rows per phase
#endif
constexpr int kSubChunks = SG_SUBCHUNKS;
constexpr int kTbLanes = SG_TB_LANES, kSubMax = SG_SUBMAX < SG_SUBCHUNKS ? SG_SUBCHUNKS : SG_SUBMAX;
constexpr int kBandSubChunks = SG_BAND_SUBCHUNKS;
// (R = 4: sweep groups are aligned to 4-column text-code words; C % 4 == 0.)

// Shared memory of one warp, in 32-bit words:
//   txt [WB/8][32] u64   text codes (1 byte per column, 4 = non-ACGT / virtual)
//   xy  [C+1][32][2]     traceback events X / Y per column, 32-bit band around
//                        the diagonal (band_base); column C = dummy
//   pm  [5][32][L]       pattern masks per code (code 4: all ones)
//   sq  [6L+4][32]       packed text (2L+1 words), pattern (2L+1), text N (L+1),
//                        pattern N (L+1) of the current segment, for traceback
template <int L> __host__ __device__ constexpr int txt_words() { return (32 * L / 4 + 2) * 32; }
template <int L> __host__ __device__ constexpr int xy_words() {
    return (KCfg<L>::C + 1) * 2 * 32;
}
template <int L> __host__ __device__ constexpr int pm_words() { return 5 * L * 32; }
// words of packed text / pattern staged per lane: the window plus the reach
// of the next window's start (W - O <= 64 for L <= 2)
template <int L> __host__ __device__ constexpr int pf_words() { return L == 1 ? 6 : L == 2 ? 10 : 12; }
template <int L> __host__ __device__ constexpr int sq_words() {
    return (2 * pf_words<L>() + 2 * (L + 1)) * 32;
}
template <int L> __host__ __device__ constexpr int warp_smem_words() {
    return txt_words<L>() + xy_words<L>() + pm_words<L>() + sq_words<L>();
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

// Shared-memory load kept in program order (issued before the arithmetic
// that follows it in the source).
__device__ __forceinline__ uint32_t lds_v(const uint32_t* p) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];"
                 : "=r"(v)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
    return v;
}

// A value the compiler cannot see through (keeps x * (1 << P) an IMAD).
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
    uint32_t r;
    asm("mov.b32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}

// x*two + b with `two` a runtime 2: an IMAD on the FMA pipe. With a literal 2
// ptxas emits LEA, which issues on the ALU pipe the bitvector logic needs.
__device__ __forceinline__ uint32_t dp_shift(uint32_t x, uint32_t two, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(two), "r"(b));
    return r;
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

// Traceback event band. Column i keeps the events of the 32 logical positions
// q in [L*P, L*P + 32), P = band_base(i): bits p in [P, P + 32/L) of every limb,
// centred on the diagonal q = i + off. Columns share P in blocks
// {4k-1 .. 4k+2} (the columns one sweep group finishes). A traceback path that
// leaves the band continues as a new segment (the suffix distances do not
// depend on where the segment starts).
template <int L> __device__ __forceinline__ int band_base(int i, int off) {
    if (L == 1) return 0;
    constexpr int SH = L == 2 ? 1 : 2;
    const int P = (((i + 1) & ~3) + off - 16) >> SH;
    return min(max(P, 0), 32 - 32 / L);
}

// The band word of a full event vector: limb r's bits p in [P, P + 32/L) at
// band bits 31 - (32/L) r - (p - P). mul = 1 << P (an IMAD per limb).
template <int L>
__device__ __forceinline__ uint32_t band_word(const uint32_t (&a)[L], uint32_t mul) {
    if constexpr (L == 1) {
        return a[0];
    } else if constexpr (L == 2) {
        return __byte_perm(a[0] * mul, a[1] * mul, 0x3276);
    } else {
        const uint32_t u = __byte_perm(a[0] * mul, a[1] * mul, 0x3700);
        const uint32_t v = __byte_perm(a[2] * mul, a[3] * mul, 0x0037);
        return __byte_perm(u, v, 0x3254);
    }
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
// (each needs only the previous step's values), giving R-way instruction-level
// parallelism instead of an R-long dependency chain per column.
// Columns >= n_w are "virtual": pattern mask all ones and boundary bits 0,
// which reproduce the init column R[n][d] exactly, so filling the wavefront
// needs no special code. The pattern masks and the traceback event
// accumulators of the R columns in flight live in rings indexed by the step at
// which row 0 entered the column; unrolling the step loop by R makes every ring
// index static (no register moves).
//
// Cell update (proj/src/dp.cpp:187-211), with c = n - i:
//   I = shl1(R[i][d-1], [c > d-1]);  D = R[i+1][d-1];  S = shl1(D, [c-1 > d-1])
//   M = shl1(R[i+1][d], [c-1 > d]) | PM[t_i];   R[i][d] = I & D & S & M
// S(i, d) equals I(i+1, d) (dp.cpp:193-194 boundary terms coincide), carried
// in ic. Traceback events of the column:
//   X |= R & ~shl1(R[i+1][d])  (D(i+1,j+1) < D(i,j));  Y |= R & ~R[i+1][d]  (D(i+1,j) < D(i,j))
template <int L, int R>
struct Sweep {
    uint32_t v[R][L];       // latest value of row r (R[col_r][d0 + r])
    uint32_t dg[R][L];      // diag input of row r at its next step
    uint32_t ic[R];         // S(col_r - 1, d) = shifted limb of I(col_r, d)
    uint32_t pmq[R][L];     // pattern mask ring
    uint32_t acc[R][2][L];  // X / Y event ring
};

// One cell of row r. bI / bM: boundary bits (0/1).
template <int L, int R, int SLOT, bool FIRST, bool CAP>
__device__ __forceinline__ void sweep_cell(Sweep<L, R>& S, int r, const uint32_t (&north)[L],
                                           uint32_t two, uint32_t bI, uint32_t bM) {
    uint32_t east[L], diag[L], I[L], M[L], Sv[L], Rv[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        east[l] = S.v[r][l];
        diag[l] = S.dg[r][l];
    }
#pragma unroll
    for (int l = 0; l + 1 < L; ++l) {
        I[l] = north[l + 1];
        M[l] = east[l + 1];
        Sv[l] = diag[l + 1];
    }
    I[L - 1] = dp_shift(north[0], two, bI);
    M[L - 1] = dp_shift(east[0], two, bM);
    Sv[L - 1] = S.ic[r];
#pragma unroll
    for (int l = 0; l < L; ++l) Rv[l] = I[l] & diag[l] & Sv[l] & (M[l] | S.pmq[SLOT][l]);
#pragma unroll
    for (int l = 0; l < L && CAP; ++l) {
        const uint32_t x = Rv[l] & ~M[l], y = Rv[l] & ~east[l];
        if (FIRST) {
            S.acc[SLOT][0][l] = x;
            S.acc[SLOT][1][l] = y;
        } else {
            S.acc[SLOT][0][l] |= x;
            S.acc[SLOT][1][l] |= y;
        }
    }
    S.ic[r] = I[L - 1];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        if (r + 1 < R) S.dg[r + 1 < R ? r + 1 : 0][l] = east[l];
        S.v[r][l] = Rv[l];
    }
}

// Rows TOP, TOP-1, ..., TOP-|Rs|+1 of step U (descending: a row reads its
// north neighbour's value from the previous step before that row updates).
template <int L, int R, int U, int TOP, bool CAP, int... Rs>
__device__ __forceinline__ void sweep_rows(Sweep<L, R>& S, const uint32_t (&t)[R + 1],
                                           uint32_t two, std::integer_sequence<int, Rs...>) {
    (sweep_cell<L, R, ((U - (TOP - Rs)) & (R - 1)), false, CAP>(S, TOP - Rs, S.v[TOP - Rs - 1],
                                                                two, t[TOP - Rs],
                                                                t[TOP - Rs + 1]),
     ...);
}

// Step U (static) of a group. SLOW: explicit boundary bits from
// g = n_w - S0 - d0 + s: row r gets [g >= 2r] (or d == 0) and [g >= 2r + 2]
// (dp.cpp:187-195 with c = n - i: [c > d-1], [c-1 > d]). Fast groups have
// every cell at least two columns from the right edge: both bits are 1.
// CAP: accumulate traceback events.
template <int L, int R, int U, bool SLOW, bool CAP>
__device__ __forceinline__ void sweep_step(Sweep<L, R>& S, const uint32_t (&north0)[L],
                                           const uint32_t (&pm0)[L], uint32_t two, uint32_t one,
                                           int g, bool z0) {
#pragma unroll
    for (int l = 0; l < L; ++l) S.pmq[U][l] = pm0[l];
    uint32_t t[R + 1];
#pragma unroll
    for (int k = 0; k <= R; ++k) t[k] = SLOW ? static_cast<uint32_t>(g >= 2 * k) : one;
    if (SLOW) t[0] |= static_cast<uint32_t>(z0);
    sweep_rows<L, R, U, R - 1, CAP>(S, t, two, std::make_integer_sequence<int, R - 1>{});
    sweep_cell<L, R, U, true, CAP>(S, 0, north0, two, t[0], t[1]);
#pragma unroll
    for (int l = 0; l < L; ++l) S.dg[0][l] = north0[l];
}

// Bit j = 0 of row r's value at column 0 (the d_opt test, dp.cpp:222).
template <int L, int R>
__device__ __forceinline__ uint32_t top_bit(const Sweep<L, R>& S, int r, int r0, int p0) {
    uint32_t v = S.v[r][0];
#pragma unroll
    for (int l = 1; l < L; ++l) v = r0 == l ? S.v[r][l] : v;
    return (v >> (31 - p0)) & 1u;
}

// Per-lane views of the warp's shared memory and parked-row scratch.
//   bnd (stride 32L words): slot c + 4 = column c (slots 0..3 pad the
//   one-group-ahead prefetch past column 0), WB + 4 = dummy store target.
//   xy (stride 64 words per column, X / Y adjacent): column C is the dummy.
//   txt: 4 text codes per word, word w + 1 = columns 4w..4w+3 (word 0 pads
//   column -1 with code 4).
template <int L>
struct LaneMem {
    uint32_t* bnd;        // + lane * L
    const uint32_t* ones;   // + lane * L: all-ones rows (R[.][-1], a window's first chunk)
    const uint32_t* zeros;  // + lane * L: all-zero rows (idle lanes)
    uint32_t* xy;         // + lane * 2
    const uint32_t* pm;   // + lane * L
    const uint32_t* txt;  // + lane
};

// Prefetch rings carried across steps and groups: the parked row for two
// steps ahead (nbr), the pattern mask of the next column (pmn) and the earlier
// chunks' events of the next finished column (ox / oy, raw).
template <int L>
struct Pref {
    uint32_t nbr[4][L];
    uint32_t pmn[L];
    uint32_t ox, oy;
};

template <int C>
__device__ __forceinline__ int xslot(int col, int n_w) {
    return col >= 0 && col < n_w && col < C ? col : C;
}

enum { kSlow = 0, kIn = 1, kOut = 2 };

// One group of R = 4 steps (static ring slots) covering row-0 columns
// col_top..col_top-3 (col_top = 3 mod 4). MODE kSlow: near the right edge
// (explicit boundary bits, virtual columns, dummy slots); kIn: every finished
// column is a real traceback-code column (static addressing); kOut: every
// cell lies right of the traceback-code region (no event capture or stores).
// DRAIN: the extra group after row 0 left column 0 (rows 1..R-1 finish; rows
// past column 0 compute harmless values on negative columns; each row's
// bit j = 0 is tested when it reaches column 0).
template <int L, int R, int C, int MODE, bool DRAIN>
__device__ __forceinline__ void sweep_group(Sweep<L, R>& S, Pref<L>& F, const LaneMem<L>& M,
                                            uint32_t codes4, uint32_t codes4n, int col_top,
                                            uint32_t two, uint32_t one, int g0, bool z0, int n_w,
                                            const uint32_t* rb, int r0, int p0, int off, int& fr,
                                            bool live) {
    static_assert(R == 4, "groups are aligned to 4-column text-code words");
    constexpr int WB = 32 * L;
    constexpr bool SLOW = MODE == kSlow, CAP = MODE != kOut;
    // group bases: row-0 parked-row slot of step 0 (read from rb: the parked
    // row, or all ones in a window's first chunk, or zeros for an idle lane),
    // finished column of step 0
    const uint32_t* nbg = rb + (col_top + 4) * 32 * L;
    const int colf0 = col_top + R - 1;
    uint32_t* pbg = M.bnd + (colf0 + 4) * 32 * L;
    uint32_t* pxg = M.xy + colf0 * 64;
    uint32_t mul = 1;
    if (CAP) {  // earlier chunks' events of step 0's finished column; band of the group
        const uint2 o = *reinterpret_cast<const uint2*>(SLOW ? M.xy + xslot<C>(colf0, n_w) * 64
                                                               : pxg);
        F.ox = o.x;
        F.oy = o.y;
        mul = opaque_u32(1u << band_base<L>(colf0, off));  // keeps band_word's x * 2^P an IMAD
    }
#define SG_STEP(U)                                                                           \
    if (!DRAIN || (U) + 1 < R) {                                                             \
        uint32_t pm0[L], north0[L];                                                          \
        _Pragma("unroll") for (int l = 0; l < L; ++l) {                                      \
            pm0[l] = F.pmn[l];                                                               \
            north0[l] = F.nbr[(U)][l];                                                       \
        }                                                                                    \
        {   /* prefetch: parked row one group ahead, pattern mask of the next column */     \
            const uint32_t* src = DRAIN ? rb : nbg - ((U) + 4) * 32 * L;                     \
            _Pragma("unroll") for (int l = 0; l < L; ++l) F.nbr[(U)][l] = src[l];            \
            const uint32_t w = (U) == 3 ? codes4n : codes4;                                  \
            const int code = static_cast<int>((w >> (8 * ((2 - (U)) & 3))) & 0xFFu);         \
            _Pragma("unroll") for (int l = 0; l < L; ++l) F.pmn[l] = M.pm[code * 32 * L + l]; \
        }                                                                                    \
        sweep_step<L, R, (U), SLOW, CAP>(S, north0, pm0, two, one, g0 + (U), z0);            \
        {   /* row R-1 finished column colf: park it, store its events */                   \
            constexpr int SL = ((U) + 1) & (R - 1);                                          \
            const int colf = colf0 - (U);                                                    \
            uint32_t* pb = pbg - (U) * 32 * L;                                               \
            uint32_t* px = pxg - (U) * 64;                                                   \
            if (SLOW) {                                                                      \
                pb = M.bnd + (colf >= 0 && colf < n_w ? colf + 4 : WB + 4) * 32 * L;         \
                px = M.xy + xslot<C>(colf, n_w) * 64;                                        \
            }                                                                                \
            if (live) /* idle lanes: the slots may hold a band-frame window's EQ */     \
                _Pragma("unroll") for (int l = 0; l < L; ++l) pb[l] = S.v[R - 1][l];         \
            if (CAP) {                                                                       \
                uint2 o;                                                                     \
                /* cleared per window; OR as an add on the FMA pipe: an event bit is set */ \
                /* by one row at most */                                    \
                o.x = dp_shift(F.ox, one, band_word<L>(S.acc[SL][0], mul));                  \
                o.y = dp_shift(F.oy, one, band_word<L>(S.acc[SL][1], mul));                  \
                *reinterpret_cast<uint2*>(px) = o;                                           \
                if ((U) + 1 < R) { /* next step's column; groups reload at their start */   \
                    const uint2 n = *reinterpret_cast<const uint2*>(                         \
                        SLOW ? M.xy + xslot<C>(colf - 1, n_w) * 64 : px - 64);               \
                    F.ox = n.x;                                                              \
                    F.oy = n.y;                                                              \
                }                                                                            \
            }                                                                                \
        }                                                                                    \
        if (DRAIN && fr < 0 && !top_bit<L, R>(S, ((U) + 1) & (R - 1), r0, p0)) fr = (U) + 1; \
    }
    SG_STEP(0) SG_STEP(1) SG_STEP(2) SG_STEP(3)
#undef SG_STEP
}

// One chunk of rows d0..d0+R-1 over columns n_w-1..0 (n_w = 0: idle lane).
// Returns the first row r of the chunk with bit j=0 of R[0][d0+r] clear, or -1.
// A lane with live == false sweeps along with all-zero rows: it produces no
// events and rewrites its stored events unchanged (its traceback is pending).
template <int L, int R, int C>
__device__ __forceinline__ int dc_chunk(int n_w, bool live, int m_w, int d0, int n_max,
                                        uint32_t two, uint32_t one, const LaneMem<L>& M) {
    constexpr int WB = 32 * L;
    static_assert(R == 4 && WB % R == 0 && C % R == 0, "R = 4 groups aligned to C");
    const uint32_t lv = live ? ~0u : 0u;
    Sweep<L, R> S;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int d = d0 + r;
#pragma unroll
        for (int l = 0; l < L; ++l) {
            S.v[r][l] = init_limb<L>(d, l) & lv;
            S.dg[r][l] = init_limb<L>(d - 1, l) & lv;
            S.pmq[r][l] = ~0u;
            S.acc[r][0][l] = S.acc[r][1][l] = 0u;
        }
        // I(n, d) = shl1(R[n][d-1], [d == 0]) with R[n][-1] = ones
        S.ic[r] = (d == 0 ? ~0u : (init_limb<L>(d - 1, 0) << 1)) & lv;
    }
    const int tsteps = ((n_max + R - 1) / R) * R;
    const int S0 = tsteps - 1;
    const bool z0 = d0 == 0 && live;
    const uint32_t* rb = !live ? M.zeros : (d0 == 0 ? M.ones : M.bnd);
    // Virtual columns >= n_w of the parked row hold R[n][d0-1].
    if (d0 > 0)
        for (int c = n_w; c <= S0; ++c)
#pragma unroll
            for (int l = 0; l < L; ++l) M.bnd[(c + 4) * 32 * L + l] = init_limb<L>(d0 - 1, l);
    Pref<L> F;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int l = 0; l < L; ++l) F.nbr[u][l] = rb[(S0 - u + 4) * 32 * L + l];
    uint32_t codes4 = M.txt[((S0 >> 2) + 1) * 32];
    {
        const int code = static_cast<int>((codes4 >> 24) & 0xFFu);  // column S0 = 3 mod 4
#pragma unroll
        for (int l = 0; l < L; ++l) F.pmn[l] = M.pm[code * 32 * L + l];
    }
    const int off = WB - m_w;
    const int r0 = off % L, p0 = off / L;
    int fr = -1;
    for (int sg = 0; sg < tsteps; sg += R) {
        const int col_top = S0 - sg;
        const uint32_t codes4n = M.txt[(col_top >> 2) * 32];  // word of column col_top - 4
        const int g0 = n_w - S0 - d0 + sg;
        int mode = kSlow;  // warp-uniform
        if (!__any_sync(kFull, n_w > 0 && g0 < 2 * R)) {
            if (col_top - R + 1 >= C) mode = kOut;
            else if (col_top + R - 1 < C) mode = kIn;
        }
        if (mode == kIn)
            sweep_group<L, R, C, kIn, false>(S, F, M, codes4, codes4n, col_top, two, one, g0, z0,
                                             n_w, rb, r0, p0, off, fr, live);
        else if (mode == kOut)
            sweep_group<L, R, C, kOut, false>(S, F, M, codes4, codes4n, col_top, two, one, g0,
                                              z0, n_w, rb, r0, p0, off, fr, live);
        else
            sweep_group<L, R, C, kSlow, false>(S, F, M, codes4, codes4n, col_top, two, one, g0,
                                               z0, n_w, rb, r0, p0, off, fr, live);
        codes4 = codes4n;
    }
    // drain: rows 1..R-1 finish (row 0 has just left column 0)
    if (!top_bit<L, R>(S, 0, r0, p0)) fr = 0;
    sweep_group<L, R, C, kSlow, true>(S, F, M, codes4, codes4, -1, two, one,
                                      n_w - S0 - d0 + tsteps, z0, n_w, rb, r0, p0, off, fr, live);
    return fr;
}

// ---------------------------------------------------------- band-frame DC (K1b)
//
// DESIGN.md §3.8. Rows are kept in DIAGONAL coordinates, one 32-bit word per
// row: bit k of a row at column i is cell (i, j = i + e_lo + k), complemented
// (bit = 1 <=> D(i, j) <= d). With e_lo = floor(d0/2) - 16 (d0 = m_w - n_w)
// the band holds every cell of every path of cost <= 30 from (0, 0) to
// (n_w, m_w): leaving it costs at least 31. Cells outside read as "D > d"
// (zeros shifted in), so rows 0..30 give D(0, 0) and every traceback decision
// exactly (DESIGN.md §3.8 has the argument). The cell update (dp.cpp:187-211 in
// these coordinates, C = ~R):
//   C[i][d] = (C[i+1][d] & EQ_i) | C[i+1][d-1] | (C[i+1][d-1] << 1) | (C[i][d-1] >> 1)
// (match, substitution, deletion, insertion). EQ_i bit k = [t_i == p_j], zero
// for j >= m_w, so the end-of-pattern column j = m_w is an ordinary band cell
// (D(i, m_w) = n_w - i) and there are no boundary bits. Traceback events:
//   X |= C[i+1][d] & ~C[i][d]          (D(i+1, j+1) < D(i, j))
//   Y |= (C[i+1][d] << 1) & ~C[i][d]   (D(i+1, j) < D(i, j))
// A cell costs 2 LOP3 + 2 FMA-pipe shifts (x * 2, mul.hi(x, 2^31) = x >> 1),
// plus 2 LOP3 where events are kept.
namespace band {
constexpr int R = 4;
constexpr int WMAX = 64;              // widest band-mode window (columns)
constexpr int CMAX = 40;              // traceback-event columns (W - O <= 40)
constexpr int kLastRow = 30;          // rows 0..30 are exact
constexpr int WARPS = 7;              // band warps per block (one block per SM) ...
constexpr int FWARPS = 0;             // (no full-frame warp in K1 mixed) ...
#ifndef SG_K0
#define SG_K0 1  // a pair whose first window fails the band frame goes to the full-frame K1
#endif
#ifndef SG_CWARPS
#define SG_CWARPS 1
#endif
constexpr int CWARPS = SG_CWARPS;             // ... plus cooperative warps
#ifndef SG_BACK_ROW
#define SG_BACK_ROW 24
#endif
#ifndef SG_COOP_SLEEP
#define SG_COOP_SLEEP 4000
#endif
constexpr int kBackRow = SG_BACK_ROW;  // a pair goes back to the band warps after D(0,0) <= 24
constexpr int kCoopSleep = SG_COOP_SLEEP;  // ns between an idle cooperative warp's polls
// per-warp shared memory, in 32-bit words:
//   eqp [WMAX + 4][32] uint2  (EQ_i, parked row) of column i at slot i + 4
//   xy  [CMAX + 2][32] uint2  parity planes (P0, P1) of columns 0..C; column C + 1
//                             (runtime) is the dummy
//   sq  packed text / pattern / N words of the window (traceback), as K1<2>
__host__ __device__ constexpr int eqp_words() { return (WMAX + 4) * 64; }
__host__ __device__ constexpr int xy_words() { return (CMAX + 2) * 64; }
}  // namespace band

// Band chunks are R = 8 rows (kBandR): eight independent cells per step, and the
// per-column work (EQ / parked-row load, park, plane update) spread over 8 cells.
constexpr int kBandR = SG_BAND_R;

template <int R>
struct BandState {
    uint32_t v[R];       // row r's latest value
    uint32_t dg[R];      // row r-1's value at row r's column + 1 (row 0: parked row)
    uint32_t dgs[R];     // dg << 1
    uint32_t eq[R];      // EQ ring: slot s % R = the column row 0 entered at step s
    uint32_t acc[R][2];  // parity planes (P0, P1) ring, same slots
};

__device__ __forceinline__ uint32_t fma_shl(uint32_t x, uint32_t two) {  // x * two (IMAD)
    uint32_t r;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(two));
    return r;
}
__device__ __forceinline__ uint32_t fma_shr(uint32_t x, uint32_t hmul) {  // x * 2^31 >> 32 (IMAD.HI)
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(hmul));
    return r;
}
// (a & b) | c | d as two LOP3s (ptxas otherwise often emits three)
__device__ __forceinline__ uint32_t or_and4(uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                            uint32_t e) {
    uint32_t t, r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(t) : "r"(a), "r"(b), "r"(c));  // (a & b) | c
    asm("lop3.b32 %0, %1, %2, %3, 0xFE;" : "=r"(r) : "r"(t), "r"(d), "r"(e));  // t | d | e
    return r;
}

// Row r's cell at step U (static). north: row r-1's value at this column.
// STD: the standard frame (bit j = cell (i, j), patterns of <= 31 bases, §3.8):
//   C[i][d] = ((C[i+1][d] >> 1) & EQ_i) | (C[i+1][d-1] >> 1) | C[i+1][d-1] | (C[i][d-1] >> 1)
// the band chunk's data flow with es = east >> 1.
template <int R, int U, int r, bool CAP, bool STD>
__device__ __forceinline__ void band_cell(BandState<R>& S, uint32_t north, uint32_t two,
                                          uint32_t hmul) {
    constexpr int SL = (U - r) & (R - 1);
    const uint32_t east = S.v[r];
    const uint32_t ns = fma_shr(north, hmul);
    const uint32_t es = STD ? fma_shr(east, hmul) : fma_shl(east, two);
    const uint32_t mt = STD ? es : east;  // the match neighbour (i+1, j+1)
    const uint32_t c = or_and4(mt, S.eq[SL], S.dg[r], S.dgs[r], ns);
    if (CAP) {
        // parity planes of the column (§3.8): P0 ^= every row, P1 ^= the odd rows
        // (d0 is a multiple of R, so row r's parity is r's). An odd row r takes
        // rows r - 1 and r into P0 (north = row r - 1 at this column).
        if (r == 1) {
            S.acc[SL][0] = north ^ c;
            S.acc[SL][1] = c;
        } else if (r & 1) {
            S.acc[SL][0] ^= north ^ c;
            S.acc[SL][1] ^= c;
        }
    }
    if (r + 1 < R) {
        S.dg[r + 1 < R ? r + 1 : 0] = east;
        S.dgs[r + 1 < R ? r + 1 : 0] = es;
    }
    S.v[r] = c;
}

enum { kBFill = 0, kBOut = 1, kBIn = 2, kBMix = 3, kBDrain = 4 };

// Lane views: eqp + lane (uint2 stride 32 per column slot), xy + lane.
struct BandMem {
    uint2* eqp;  // slot(col) = col + 4
    uint2* xy;   // column c at xy[c * 32]
};

template <int R, int MODE, int U, bool STD, int r>
__device__ __forceinline__ void band_rows(BandState<R>& S, uint32_t two, uint32_t hmul) {
    // rows R-1..1, descending: a row reads its upper row's value before it updates
    if constexpr (r >= 1) {
        if constexpr ((MODE == kBFill && r <= U) || (MODE == kBDrain && r > U) ||
                      (MODE != kBFill && MODE != kBDrain))
            band_cell<R, U, r, MODE != kBOut, STD>(S, S.v[r - 1], two, hmul);
        band_rows<R, MODE, U, STD, r - 1>(S, two, hmul);
    }
}

// Step U of a group of R steps. Row 0 works on columns col_top .. col_top - R + 1;
// row r lags r columns. MODE: kBFill (rows r <= U start at column W-1), kBDrain
// (rows r > U finish at column 0), kBOut (no plane columns), kBIn (every column
// the last row finishes keeps its planes), kBMix (stores of columns >= C go to the
// dummy). F: (EQ, parked row) of row 0's column, loaded four steps ahead.
template <int R, int MODE, int U, bool STD>
__device__ __forceinline__ void band_step(BandState<R>& S, uint2 (&F)[4], const BandMem& M,
                                          int col_top, int C, uint32_t two,
                                          uint32_t hmul, uint32_t two_l, uint32_t hmul_l,
                                          uint32_t one_l, bool live) {
    constexpr bool CAP = MODE != kBOut;
    constexpr bool LAST = (MODE == kBFill ? U == R - 1 : true) && (MODE != kBDrain || U < R - 1);
    constexpr bool STORE_EV = CAP && LAST;
    const int cl = col_top - U + R - 1;  // the column the last row finishes at this step
    uint2* px = M.xy + (MODE == kBIn ? cl : (cl < C ? cl : C)) * 32;
    uint2 old = make_uint2(0u, 0u);
    if (STORE_EV) old = *px;
    const uint2 f = F[U & 3];
    band_rows<R, MODE, U, STD, R - 1>(S, two, hmul);
    if (MODE != kBDrain) {  // row 0: north = parked row of this column, masked for idle lanes
        S.eq[U] = f.x;
        band_cell<R, U, 0, CAP, STD>(S, f.y, two, hmul_l);
        // (right of the plane columns the FMA pipe is the busier one: AND there)
        S.dg[0] = MODE == kBOut ? f.y & (0u - one_l) : fma_shl(f.y, one_l);
        S.dgs[0] = STD ? fma_shr(f.y, hmul_l) : fma_shl(f.y, two_l);
        // row 0's column four steps on, into the registers f just left
        F[U & 3] = M.eqp[(col_top - U - 4 + 4) * 32];
    }
    if (LAST) {
        // park the last row (idle lanes do not)
        if (live) reinterpret_cast<uint32_t*>(M.eqp + (cl + 4) * 32)[1] = S.v[R - 1];
        if (STORE_EV) {
            // the planes of a window start at zero (load_segment) and XOR over its
            // chunks; an idle lane's all-zero rows leave them unchanged
            constexpr int SLL = (U + 1) & (R - 1);
            *px = make_uint2(old.x ^ S.acc[SLL][0], old.y ^ S.acc[SLL][1]);
        }
    }
}

template <int R, int MODE, bool STD, int U = 0>
__device__ __forceinline__ void band_group(BandState<R>& S, uint2 (&F)[4], const BandMem& M,
                                           int col_top, int C, uint32_t two,
                                           uint32_t hmul, uint32_t two_l, uint32_t hmul_l,
                                           uint32_t one_l, bool live) {
    if constexpr (U < R) {
        band_step<R, MODE, U, STD>(S, F, M, col_top, C, two, hmul, two_l, hmul_l, one_l, live);
        band_group<R, MODE, STD, U + 1>(S, F, M, col_top, C, two, hmul, two_l, hmul_l, one_l, live);
    }
}

// init column (i = n_w) of row d: bits k in [K0 - d, K0] (D(n, j) = m - j <= d)
__device__ __forceinline__ uint32_t band_init(int d, int K0) {
    if (d < 0) return 0u;
    const int lo = max(K0 - d, 0);
    return (0xFFFFFFFFu >> (31 - K0)) & (0xFFFFFFFFu << lo);
}

// One chunk of rows d0..d0+R-1 over the W columns (W % R == 0) of a band window.
// Returns the first row r with D(0, 0) <= d0 + r, or -1. Idle lanes (live = false)
// run on all-zero rows: they keep their stored planes and do not park.
template <int R, bool STD>
__device__ __forceinline__ int band_chunk(bool live, int d0, int W, int C, int K0, int k00,
                                          const BandMem& M, uint32_t two, uint32_t hmul) {
    const uint32_t lv = live ? ~0u : 0u;
    BandState<R> S;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        S.v[r] = band_init(d0 + r, K0) & lv;
        S.dg[r] = band_init(d0 + r - 1, K0) & lv;
        S.dgs[r] = STD ? S.dg[r] >> 1 : S.dg[r] << 1;
        S.eq[r] = 0u;
        S.acc[r][0] = S.acc[r][1] = 0u;
    }
    const uint32_t two_l = two & lv, hmul_l = hmul & lv, one_l = (two >> 1) & lv;
    uint2 F[4];
#pragma unroll
    for (int U = 0; U < 4; ++U) F[U] = M.eqp[(W - 1 - U + 4) * 32];
    band_group<R, kBFill, STD>(S, F, M, W - 1, C, two, hmul, two_l, hmul_l, one_l, live);
    // steady groups in three runs (no per-group mode test): right of the plane
    // columns, the groups that straddle column C, inside them
    int col_top = W - 1 - R;
    for (; col_top >= R - 1 && col_top - (R - 1) >= C; col_top -= R)
        band_group<R, kBOut, STD>(S, F, M, col_top, C, two, hmul, two_l, hmul_l, one_l, live);
    for (; col_top >= R - 1 && col_top + R - 1 >= C; col_top -= R)
        band_group<R, kBMix, STD>(S, F, M, col_top, C, two, hmul, two_l, hmul_l, one_l, live);
    for (; col_top >= R - 1; col_top -= R)
        band_group<R, kBIn, STD>(S, F, M, col_top, C, two, hmul, two_l, hmul_l, one_l, live);
    band_group<R, kBDrain, STD>(S, F, M, -1, C, two, hmul, two_l, hmul_l, one_l, live);
    int fr = -1;
#pragma unroll
    for (int r = R - 1; r >= 0; --r)
        if ((S.v[r] >> k00) & 1u) fr = r;
    return fr;
}

// ------------------------------------------------------------------ K1

// Shared memory words of one K1 warp (BAND: the band-frame layout, §3.8).
template <int L, bool BAND> __host__ __device__ constexpr int k1_warp_words() {
    // band: rings of 8 packed words per side plus the N words (sq_words<2> with PFW 8)
    return BAND ? band::eqp_words() + band::xy_words() + (2 * 8 + 2 * (L + 1)) * 32
                : warp_smem_words<L>();
}
// Hand-over queues between band and full-frame warps (K1 mixed, §3.8): a ring
// of pair ids, q[0] = head, q[1] = tail, slots q[32 + k % cap] hold pair + 1
// (0 = empty). The pair's state is written before the slot is published.
__device__ __forceinline__ void q_push(uint32_t* q, int cap, int pair) {
    __threadfence();
    const unsigned t = atomicAdd(q + 1, 1u);
    uint32_t* slot = q + 32 + t % static_cast<unsigned>(cap);
    while (atomicCAS(slot, 0u, static_cast<uint32_t>(pair) + 1u) != 0u) __nanosleep(200);
}
__device__ __forceinline__ int q_pop(uint32_t* q, int cap) {
    const unsigned h = *reinterpret_cast<volatile unsigned*>(q);
    const unsigned t = *reinterpret_cast<volatile unsigned*>(q + 1);
    if (static_cast<int>(t - h) <= 0) return -1;
    if (atomicCAS(q, h, h + 1u) != h) return -1;  // another lane took it: retry later
    uint32_t* slot = q + 32 + h % static_cast<unsigned>(cap);
    uint32_t v;
    while ((v = atomicExch(slot, 0u)) == 0u) __nanosleep(200);  // reserved, not yet written
    __threadfence();
    return static_cast<int>(v) - 1;
}

// Pops up to `maxn` entries with one CAS (a cooperative warp takes several when
// the queue is long: one CAS per pair serialises the pops on one L2 line when
// every pair hands its last window over at once). Single-thread.
__device__ __forceinline__ int q_pop_n(uint32_t* q, int cap, int maxn, int* out) {
    const unsigned h = *reinterpret_cast<volatile unsigned*>(q);
    const unsigned t = *reinterpret_cast<volatile unsigned*>(q + 1);
    const int avail = static_cast<int>(t - h);
    if (avail <= 0) return 0;
    const int take = min(maxn, max(1, avail / 32));
    if (atomicCAS(q, h, h + static_cast<unsigned>(take)) != h) return 0;
    for (int k = 0; k < take; ++k) {
        uint32_t* slot = q + 32 + (h + k) % static_cast<unsigned>(cap);
        uint32_t v;
        while ((v = atomicExch(slot, 0u)) == 0u) __nanosleep(200);
        out[k] = static_cast<int>(v) - 1;
    }
    __threadfence();
    return take;
}

// Idle wait of at least `cycles` SM cycles (a single nanosleep can return after
// a fraction of its argument; an idle warp's polls take issue slots and L2
// bandwidth from the working warps).
__device__ __forceinline__ void idle_wait(long long cycles) {
    const long long t0 = clock64();
    do {
        __nanosleep(1000);
    } while (clock64() - t0 < cycles);
}

// Warp-aggregated pop for the calling lanes that `want` a pair: one CAS on the
// head claims up to one entry per such lane (a per-lane CAS serialises every pop
// on one address).
__device__ __forceinline__ int q_pop_warp(uint32_t* q, int cap, bool want) {
    const unsigned active = __activemask();
    const unsigned wm = __ballot_sync(active, want);
    if (!want) return -1;
    const int leader = __ffs(wm) - 1;
    const int lane = threadIdx.x & 31;
    unsigned h = 0, take = 0;
    if (lane == leader) {
        h = *reinterpret_cast<volatile unsigned*>(q);
        const unsigned t = *reinterpret_cast<volatile unsigned*>(q + 1);
        const int avail = static_cast<int>(t - h);
        take = avail > 0 ? min(static_cast<unsigned>(avail), static_cast<unsigned>(__popc(wm))) : 0u;
        if (take && atomicCAS(q, h, h + take) != h) take = 0;  // lost the race: retry later
    }
    h = __shfl_sync(wm, h, leader);
    take = __shfl_sync(wm, take, leader);
    const unsigned rank = __popc(wm & ((1u << lane) - 1u));
    if (rank >= take) return -1;
    uint32_t* slot = q + 32 + (h + rank) % static_cast<unsigned>(cap);
    uint32_t v;
    while ((v = atomicExch(slot, 0u)) == 0u) __nanosleep(200);  // reserved, not yet written
    __threadfence();
    return static_cast<int>(v) - 1;
}

// K1 mixed's lists of pairs it leaves to the launches after it (the tail K1's t_list,
// the full-frame K1's u_list). Pipelined launches (P.body_done) keep
// one list and one count per output slice — slice sl's region starts at entry sl *
// slice_pairs, the last slice takes the rest of the pairs — and count the pairs of
// each slice that have left the mixed kernel:
// the slice's tail K1 starts once its count is complete (k1_tail's wait).
__device__ __forceinline__ void body_left(const AlignParams& P, int pair) {
    if (!P.body_done) return;
    __threadfence();  // the pair's state and its list entry before the count
    atomicAdd(P.body_done + min(pair / P.slice_pairs, P.last_slice), 1u);
}
__device__ __forceinline__ void list_push(const AlignParams& P, bool tail, int pair) {
    const int sl = P.body_done ? min(pair / P.slice_pairs, P.last_slice) : 0;
    int32_t* const list = (tail ? P.t_list : P.u_list) +
                          (P.body_done ? static_cast<long long>(sl) * P.slice_pairs : 0ll);
    list[atomicAdd((tail ? P.t_count : P.u_count) + sl, 1u)] = pair;
    body_left(P, pair);
}

// The K1 window loop of one warp. BAND = true: the band frame (K1b) — windows
// it cannot take (final windows, n_w < W, |m_w - n_w| > 30, D(0, 0) > 30) go
// with the pair to a full-frame warp (P.mixed); a full-frame warp hands the
// pair back once its next window is a band window again.
template <int L, bool BAND, bool TAIL = false>
__device__ __forceinline__ void k1_body(const AlignParams& P, uint32_t* const wbase,
                                        const long long gwarp, uint32_t* const bnd_smem,
                                        uint32_t* const eqp_smem) {
    static_assert(!BAND || L == 2, "the band pass stages sequences as K1<2>");
    constexpr int R = KCfg<L>::R, C = KCfg<L>::C, WB = 32 * L, NW = 2 * L;
    const int lane = threadIdx.x & 31;
    uint64_t* const txt = reinterpret_cast<uint64_t*>(wbase);   // [WB/8][32]
    uint32_t* const xy = BAND ? wbase + band::eqp_words()       // band: [CMAX+1][32][2]
                              : wbase + txt_words<L>();         // [C+1][32][2]
    uint32_t* const pmv = xy + xy_words<L>();                    // [5][32][L]
    uint32_t* const sq = BAND ? xy + band::xy_words() : pmv + pm_words<L>();  // [6L+4][32]
    // band warps: (EQ, parked row) at the start of the warp's memory; full-frame
    // warps of the mixed kernel: STD windows use the parked-row region
    const BandMem bmem{reinterpret_cast<uint2*>(BAND ? wbase : eqp_smem) + lane,
                       reinterpret_cast<uint2*>(xy) + lane};
    // band warps stage each side's packed words in a ring of 8 (the window needs 6;
    // the next one starts <= 3 words on) refilled from 3 prefetched words
    constexpr int PFW = BAND ? 8 : pf_words<L>();
    constexpr int NXW = BAND ? 3 : PFW;
    uint32_t* const sq_t = sq;                                   // text staging (PFW words)
    uint32_t* const sq_p = sq + PFW * 32;                        // pattern staging (PFW)
    uint32_t* const sq_tn = sq + 2 * PFW * 32;                   // text N words (L+1)
    uint32_t* const sq_pn = sq + (2 * PFW + L + 1) * 32;         // pattern N words (L+1)
    // parked rows [WB+5][32][L]: in shared memory for the mixed kernel's full-frame warp
    uint32_t* const bnd = bnd_smem ? bnd_smem : P.bnd + gwarp * (WB + 5) * 32 * L;
    const uint32_t two = static_cast<uint32_t>(P.two), one = two >> 1;
    const LaneMem<L> lmem{bnd + lane * L, P.bnd_ones + lane * L, P.bnd_zeros + lane * L,
                          xy + lane * 2, pmv + lane * L,
                          reinterpret_cast<const uint32_t*>(txt) + lane};

    if (!BAND) {
#pragma unroll
        for (int l = 0; l < L; ++l) pmv[(4 * 32 + lane) * L + l] = ~0u;  // non-ACGT text
#pragma unroll
        for (int b = 0; b <= WB / 4; ++b)  // idle lanes and the column -1 pad: code 4
            reinterpret_cast<uint32_t*>(txt)[b * 32 + lane] = 0x04040404u;
    }

    const int W = P.W;
    const int step_limit = W - P.O;
    const int K = P.single ? P.k_single : W;  // edit budget: rows 0..K
    // fresh pairs of this launch (a device count when a pre-pass split the batch)
    // (read through L2: a pipelined launch's count was written by K1 mixed running beside it)
    int n_fresh = P.n_pairs;
    if (P.n_fresh) n_fresh = __ldcg(P.n_fresh);
    // band pass: traceback-event columns, last exact row, shift multipliers
    const int cmax = BAND ? step_limit : C;
    const int band_last = min(K, band::kLastRow);
    // band chunks per phase: kBandSubChunks (16 rows) unless the host expects windows of
    // a few edits (cfg2, cfg4 W = 32: one 8-row chunk solves nearly every window, and a
    // second one would run for the whole warp whenever one lane needs it)
    const int band_sub = P.band_subchunks > 0 ? P.band_subchunks : kBandSubChunks;
    const uint32_t hmul = two << 30;  // 2^31 at run time: mul.hi(x, hmul) = x >> 1

    // ---- lane state ----
    int pair = -1;
    int n_tot = 0, m_tot = 0;
    int64_t tbase = 0, pbase = 0;
    bool hasn = false;
    int toff = 0, poff = 0, n_w = 0, m_w = 0, limit = 0;
    bool first_seg = true;
    int d0 = 0, found_d = -1, expect_d = -1;
    int dist = 0, nwin = 0, status = 0;
    int window_cap = 0;
    int e_lo = 0, K0 = 0;  // band window: bit k <-> j = i + e_lo + k; (n_w, m_w) at bit K0
    int pass_win = 0;      // windows this warp completed for the pair (hand-back after one)
    int last_d = 0;        // D(0, 0) of the last window
    unsigned long long ph_fresh_end = 0;  // diagnostics: when the fresh pairs ran out
    bool defer_now = false;
    bool std_win = false;  // full-frame warp, mixed: the window runs in the STD frame (m_w <= 31)
    int hand_to = 0;       // mixed: the role the pair goes to (0 band, 1 full frame, 2 cooperative)
    // Sequence staging: sq_t / sq_p hold PFW packed words from word st_tw / st_pw;
    // the segment's text / pattern start at base t_sh / p_sh inside them. The
    // words of the region the next window can start in are prefetched into
    // registers (nx_t / nx_p) while the current window runs.
    uint32_t nx_t[NXW], nx_p[NXW];
    int64_t nx_tw = -1, nx_pw = -1;  // band: one past the last staged word (-1: none)
    int64_t pf_tw = -1, pf_pw = -1;  // band: first word in nx_t / nx_p
    int t_sh = 0, p_sh = 0;
    int tb0 = 0, pb0 = 0;            // band: ring slot of the window's first word
    // output
    uint32_t* outw = nullptr;
    int out_bytes = 0, cur_op = -1, cur_len = 0, acc_n = 0;
    uint32_t acc = 0;
    // counters (InstrumentationCounters, proj/include/scrooge/dp.hpp:46-66)
    unsigned long long c_stored = 0, c_writes = 0, c_reads = 0, c_rows = 0, c_cells = 0,
                       c_bequiv = 0;

    // CIGAR runs (cigar_append, proj/src/cigar.cpp:9-16) as bytes
    // (op << 6) | (len - 1): the open byte is (cur_op, cur_len <= 64); it is
    // written when the op changes or it is full, so a run of length n becomes
    // ceil(n / 64) bytes (consecutive same-op bytes continue one run).
    auto put_byte = [&](uint32_t b) {
        acc |= b << (8 * acc_n);
        ++out_bytes;
        if (++acc_n == 4) {
            *outw++ = acc;
            acc = 0;
            acc_n = 0;
        }
    };
    auto emit = [&](int op, int len) {  // len >= 1
        if (op == cur_op && cur_len + len <= 64) {
            cur_len += len;
            return;
        }
        if (op == cur_op) {
            len -= 64 - cur_len;
            cur_len = 64;
        }
        if (cur_op >= 0) put_byte((static_cast<uint32_t>(cur_op) << 6) | (cur_len - 1));
        while (len > 64) {
            put_byte((static_cast<uint32_t>(op) << 6) | 63u);
            len -= 64;
        }
        cur_op = op;
        cur_len = len;
    };

    // Pattern masks, text codes and packed sequences of the current segment.
    auto load_segment = [&]() {
        const int off = WB - m_w;
        // Sequence words load through L2 only (ld.global.cg): with a streamed
        // upload a line read early into L1 could hold words of a chunk that had
        // not arrived yet (the staging reads run past the pair's end).
        uint32_t pw[NW + 1], pn[L + 1], tw[NW + 1], tn[L + 1];
        if constexpr (BAND) {
            const int64_t ta = tbase + toff, pa = pbase + poff;
            const int64_t wt = ta >> 4, wp = pa >> 4;
            auto stage = [&](uint32_t* ring, uint32_t (&nx)[NXW], int64_t& hi, int64_t& pf,
                             int64_t w0) {
                const int64_t need = w0 + 6;
                if (hi < 0 || w0 < hi - 6 || need > hi + 3) {  // a new pair (or a jump)
#pragma unroll
                    for (int k = 0; k < 6; ++k)
                        ring[((w0 + k) & 7) * 32 + lane] = __ldcg(P.seq + w0 + k);
                    hi = need;
                } else {
                    const bool have = pf == hi;
#pragma unroll
                    for (int k = 0; k < 3; ++k)
                        if (hi + k < need)
                            ring[((hi + k) & 7) * 32 + lane] = have ? nx[k] : __ldcg(P.seq + hi + k);
                    hi = max(hi, need);
                }
                // the words the next window can add (it starts <= 3 words on), issued
                // here (volatile: not sunk towards their use a phase later)
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(nx[k]) : "l"(P.seq + hi + k));
                pf = hi;
            };
            stage(sq_t, nx_t, nx_tw, pf_tw, wt);
            stage(sq_p, nx_p, nx_pw, pf_pw, wp);
            t_sh = static_cast<int>(ta - 16 * wt);
            p_sh = static_cast<int>(pa - 16 * wp);
            tb0 = static_cast<int>(wt & 7);
            pb0 = static_cast<int>(wp & 7);
#pragma unroll
            for (int k = 0; k <= NW; ++k) {
                tw[k] = __funnelshift_r(sq_t[((tb0 + k) & 7) * 32 + lane],
                                        sq_t[((tb0 + k + 1) & 7) * 32 + lane], 2 * t_sh);
                pw[k] = __funnelshift_r(sq_p[((pb0 + k) & 7) * 32 + lane],
                                        sq_p[((pb0 + k + 1) & 7) * 32 + lane], 2 * p_sh);
            }
        } else {
            const int64_t ta = tbase + toff, pa = pbase + poff;
            const int64_t wt = ta >> 4, wp = pa >> 4;
            // prefetched region usable? (it covers [16 nx_w, 16 (nx_w + PFW)))
            const bool hit_t = nx_tw >= 0 && wt >= nx_tw && wt + NW + 1 < nx_tw + PFW;
            const bool hit_p = nx_pw >= 0 && wp >= nx_pw && wp + NW + 1 < nx_pw + PFW;
            if (!hit_t) {
                nx_tw = wt;
#pragma unroll
                for (int k = 0; k < PFW; ++k) nx_t[k] = __ldcg(P.seq + wt + k);
            }
            if (!hit_p) {
                nx_pw = wp;
#pragma unroll
                for (int k = 0; k < PFW; ++k) nx_p[k] = __ldcg(P.seq + wp + k);
            }
#pragma unroll
            for (int k = 0; k < PFW; ++k) {
                sq_t[k * 32 + lane] = nx_t[k];
                sq_p[k * 32 + lane] = nx_p[k];
            }
            t_sh = static_cast<int>(ta - 16 * nx_tw);
            p_sh = static_cast<int>(pa - 16 * nx_pw);
#pragma unroll
            for (int k = 0; k <= NW; ++k) {
                const int bt = t_sh + 16 * k, bp = p_sh + 16 * k;
                tw[k] = __funnelshift_r(sq_t[(bt >> 4) * 32 + lane],
                                        sq_t[((bt >> 4) + 1) * 32 + lane], 2 * (bt & 15));
                pw[k] = __funnelshift_r(sq_p[(bp >> 4) * 32 + lane],
                                        sq_p[((bp >> 4) + 1) * 32 + lane], 2 * (bp & 15));
            }
            // prefetch the region of the next window (starts <= W - O further on)
            nx_tw = wt;
            nx_pw = wp;
#pragma unroll
            for (int k = 0; k < PFW; ++k) {
                nx_t[k] = __ldcg(P.seq + wt + k);
                nx_p[k] = __ldcg(P.seq + wp + k);
            }
        }
#pragma unroll
        for (int l = 0; l <= L; ++l) pn[l] = tn[l] = 0;
        if (hasn) {
            load_bits<L + 1>(P.nmask, pbase + poff, pn);
            load_bits<L + 1>(P.nmask, tbase + toff, tn);
        }
        if ((!BAND || TAIL) && std_win) {
            // (§3.8) STD frame: EQ_i = plane t_i of the pattern, bits j < m_w <= 31;
            // the planes go to this lane's event columns 0..3 (dead until the first
            // chunk overwrites them), the parked row starts as row -1 (zeros)
            const uint32_t lo = compress_stride<2>(pw[0] & 0x55555555u) |
                                (compress_stride<2>(pw[1] & 0x55555555u) << 16);
            const uint32_t hi = compress_stride<2>((pw[0] >> 1) & 0x55555555u) |
                                (compress_stride<2>((pw[1] >> 1) & 0x55555555u) << 16);
            const uint32_t valid = ((1u << m_w) - 1u) & ~pn[0];
            uint32_t* const pl = xy + lane * 2;  // column c at pl[c * 64]
            pl[0 * 64] = ~lo & ~hi & valid;
            pl[1 * 64] = lo & ~hi & valid;
            pl[2 * 64] = ~lo & hi & valid;
            pl[3 * 64] = lo & hi & valid;
#pragma unroll
            for (int k = 0; k < NW; ++k) {  // (static k: tw[] stays in registers)
                if (16 * k >= n_w) break;
                const int bt = t_sh + 16 * k;
                const uint32_t tword = BAND ? tw[k]
                                            : __funnelshift_r(sq_t[(bt >> 4) * 32 + lane],
                                                              sq_t[((bt >> 4) + 1) * 32 + lane],
                                                              2 * (bt & 15));
                const uint32_t tnw = hasn ? tn[k >> 1] >> (16 * (k & 1)) : 0u;
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int code = static_cast<int>((tword >> (2 * u)) & 3u);
                    uint32_t e = pl[code * 64];
                    if (hasn && ((tnw >> u) & 1u)) e = 0u;  // non-ACGT text matches nothing
                    bmem.eqp[(16 * k + u + 4) * 32] = make_uint2(e, 0u);
                }
            }
            for (int c = 0; c <= cmax; ++c) bmem.xy[c * 32] = make_uint2(0u, 0u);  // planes start at 0
#pragma unroll
            for (int k = 0; k <= L; ++k) {
                sq_tn[k * 32 + lane] = tn[k];
                sq_pn[k * 32 + lane] = pn[k];
            }
            return;
        }
        if constexpr (BAND) {
            // (§3.8) code planes of the pattern over j in [-32, 96) as (word w, word
            // w + 1) pairs, w = 0..2, one uint2 per (code, w) in this lane's event
            // columns 0..14 (dead until the window's first chunk overwrites them);
            // code 4 (non-ACGT text) matches nothing
            uint32_t plo[2], phi[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                plo[h] = compress_stride<2>(pw[2 * h] & 0x55555555u) |
                         (compress_stride<2>(pw[2 * h + 1] & 0x55555555u) << 16);
                phi[h] = compress_stride<2>((pw[2 * h] >> 1) & 0x55555555u) |
                         (compress_stride<2>((pw[2 * h + 1] >> 1) & 0x55555555u) << 16);
            }
            // per code c (and c | 4 for a non-ACGT text base: no match), the plane
            // over j in [e_lo, e_lo + 96) as (s0, s1), (s1, s2) pairs: column i's
            // window is then bits [i, i + 32) of s, a static funnel shift
            uint2* const lut = bmem.xy;  // entry (2c + w) at lut[(2c + w) * 32], c < 8
            const int ob = e_lo + 32;    // j = e_lo is bit ob of the [-32, 96) plane
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t q[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int vb = min(max(m_w - 32 * h, 0), 32);
                    const uint32_t valid = (vb == 32 ? ~0u : ((1u << vb) - 1u)) & ~pn[h];
                    const uint32_t lo = plo[h], hi = phi[h];
                    const uint32_t e = c == 0 ? ~lo & ~hi : c == 1 ? lo & ~hi
                                       : c == 2 ? ~lo & hi : lo & hi;
                    q[h + 1] = e & valid;  // j >= m_w and pattern N: no match
                }
                const uint32_t s0 = __funnelshift_r(q[0], q[1], ob);
                const uint32_t s1 = __funnelshift_r(q[1], q[2], ob);
                const uint32_t s2 = __funnelshift_r(q[2], q[3], ob);
                lut[(2 * c) * 32] = make_uint2(s0, s1);
                lut[(2 * c + 1) * 32] = make_uint2(s1, s2);
                lut[(2 * c + 8) * 32] = make_uint2(0u, 0u);  // code c | 4
                lut[(2 * c + 9) * 32] = make_uint2(0u, 0u);
            }
            // EQ_i of every column (the parked row starts as row -1: zeros); the N
            // bits only where a lane of the warp has a non-ACGT base
            if (__any_sync(__activemask(), hasn)) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (16 * k >= n_w) break;
                    const uint32_t tword = tw[k];
                    const uint32_t tnw = hasn ? tn[k >> 1] >> (16 * (k & 1)) : 0u;
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        const int i = 16 * k + u;
                        const uint32_t code = ((tword >> (2 * u)) & 3u) | (((tnw >> u) & 1u) << 2);
                        const uint2 pr = lut[(2 * code + (i >> 5)) * 32];
                        bmem.eqp[(i + 4) * 32] = make_uint2(__funnelshift_r(pr.x, pr.y, i & 31), 0u);
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (16 * k >= n_w) break;
                    const uint32_t tword = tw[k];
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        const int i = 16 * k + u;
                        const uint2 pr = lut[(2 * ((tword >> (2 * u)) & 3u) + (i >> 5)) * 32];
                        bmem.eqp[(i + 4) * 32] = make_uint2(__funnelshift_r(pr.x, pr.y, i & 31), 0u);
                    }
                }
            }
            // the parity planes of the window start at zero (the LUT above is dead)
            for (int c = 0; c <= cmax; ++c) bmem.xy[c * 32] = make_uint2(0u, 0u);
#pragma unroll
            for (int k = 0; k <= L; ++k) {
                sq_tn[k * 32 + lane] = tn[k];
                sq_pn[k * 32 + lane] = pn[k];
            }
            return;
        }
        uint32_t pwl[NW], pnl[L];
#pragma unroll
        for (int k = 0; k < NW; ++k) pwl[k] = pw[k];
#pragma unroll
        for (int k = 0; k < L; ++k) pnl[k] = pn[k];
#pragma unroll
        for (int r = 0; r < L; ++r) {
            const int rho = class_of<L>(r, off);
            const uint32_t lo = limbify<L>(gather_codes<L>(pwl, rho, 0), r, off, rho);
            const uint32_t hi = limbify<L>(gather_codes<L>(pwl, rho, 1), r, off, rho);
            const uint32_t nn = hasn ? limbify<L>(gather_bits<L>(pnl, rho), r, off, rho) : 0u;
            // PM[c] bit = 0 iff pattern base == c (proj/src/dp.cpp:8-21); N matches nothing
            pmv[(0 * 32 + lane) * L + r] = lo | hi | nn;
            pmv[(1 * 32 + lane) * L + r] = ~lo | hi | nn;
            pmv[(2 * 32 + lane) * L + r] = lo | ~hi | nn;
            pmv[(3 * 32 + lane) * L + r] = ~lo | ~hi | nn;
        }
        // text codes as bytes, 8 columns per u64 (non-ACGT -> 4); columns >= n_w
        // are mapped to code 4 by the sweep itself
        uint32_t* const txt32 = reinterpret_cast<uint32_t*>(txt);
#pragma unroll
        for (int h = 0; h < WB / 4; ++h) {  // word h + 1: columns 4h..4h+3
            uint32_t c = spread4(tw[h >> 2] >> (8 * (h & 3)));
            if (hasn) {
                const uint32_t nm = spread4bits(tn[h >> 3] >> (4 * (h & 7))) * 0xFFu;
                c = (c & ~nm) | (0x04040404u & nm);
            }
            // columns >= n_w are virtual: code 4 (all-ones mask)
            const int valid = n_w - 4 * h;
            if (valid < 4) c = valid <= 0 ? 0x04040404u : (c & (0xFFFFFFFFu >> (8 * (4 - valid))))
                                                          | (0x04040404u << (8 * valid));
            txt32[(h + 1) * 32 + lane] = c;
        }
        // the segment's traceback events start empty (chunks OR into them)
#pragma unroll 4
        for (int c = 0; c <= C; ++c) *reinterpret_cast<uint2*>(xy + c * 64 + lane * 2) = make_uint2(0u, 0u);
        // N words of the segment for the traceback's match runs
#pragma unroll
        for (int k = 0; k <= L; ++k) {
            sq_tn[k * 32 + lane] = tn[k];
            sq_pn[k * 32 + lane] = pn[k];
        }
    };

    // Geometry of the next logical window of the current pair
    // (aligner.cpp:44-64). Returns 0 when the pair is complete (residues
    // appended), 1 for a window, 2 when the pair goes to another warp role (the
    // queue in hand_to) before this window.
    auto next_window = [&]() -> int {
        const int n_rem = n_tot - toff, m_rem = m_tot - poff;
        if (n_rem == 0 || m_rem == 0) {
            if (n_rem + m_rem > 0) {  // aligner.cpp:48-57
                emit(n_rem == 0 ? 2 : 3, n_rem + m_rem);
                dist += n_rem + m_rem;
            }
            return 0;
        }
        // single-window mode (aligner.cpp:87-112): the whole pair is one final window
        const bool fin = P.single || (n_rem <= W && m_rem <= W);
        n_w = P.single ? n_rem : min(W, n_rem);
        m_w = P.single ? m_rem : min(W, m_rem);
        {
            const int dl = m_w - n_w;
            const bool band_ok = !fin && n_w == W && dl <= band::kLastRow && dl >= -band::kLastRow;
            // full-width non-final windows the single-word frames cannot take go
            // to a cooperative warp (§3.9)
            const bool wide_ok = !fin && n_w == W && m_w >= 32;
            const bool std_ok = !fin && n_w == W && m_w <= 31;  // the STD frame takes it
            std_win = false;
            if (TAIL) {
                // the tail K1 takes STD windows only; the rest of the pair goes on
                // to the full-frame K1
                if (!std_ok) {
                    hand_to = 4;
                    return 2;
                }
                std_win = true;
            } else if (BAND) {
                // a window the STD frame takes never runs in the band frame: STD is
                // exact for every row (a band failure would otherwise come back here)
                if (!band_ok || std_ok) {
                    // the pair's tail: an STD window (m_w <= 31) goes to the tail K1, a
                    // final window to the full-frame K1 after it; any other window (|m_w
                    // - n_w| > 30, a text or pattern all but consumed) to a cooperative
                    // warp, which hands an STD window on to the tail K1
                    hand_to = std_ok && P.t_list ? 5 : fin && P.u_list ? 4 : 2;
                    return 2;
                } else {
                    e_lo = (dl >> 1) - 16;
                    K0 = dl - e_lo;
                }
            } else if (P.mixed && band_ok && pass_win > 0 && last_d <= band::kBackRow) {
                hand_to = 0;
                return 2;  // back on track: the band frame takes the pair again
            } else if (P.mixed && wide_ok) {
                hand_to = 2;
                return 2;
            } else {
                std_win = bnd_smem != nullptr && std_ok;
            }
        }
        limit = fin ? -1 : step_limit;
        first_seg = true;
        d0 = 0;
        found_d = -1;
        expect_d = -1;
        return 1;
    };

    // Hand the pair to the next pass (the other frame) before its current window.
    auto defer_pair = [&]() {
        P.distance[pair] = dist;
        P.windows[pair] = nwin;
        P.status[pair] = 0;
        P.out_bytes[pair] = out_bytes;
        if (P.counters) {
            uint64_t* c = P.counters + 7ll * pair;
            c[0] = c_stored;
            c[1] = c_writes;
            c[2] = c_reads;
            c[3] = c_rows;
            c[4] = c_cells;
            c[6] = c_bequiv;
        }
        int32_t* rs = P.resume_state + 4ll * pair;
        rs[0] = toff;
        rs[1] = poff;
        rs[2] = (cur_op & 0xFF) | (cur_len << 8);
        rs[3] = static_cast<int32_t>(acc);
        if (BAND && hand_to == 5) {  // the tail K1 resumes the pair (its STD window)
            list_push(P, true, pair);
            if (P.mixed) atomicSub(P.remaining, 1u);
            return;
        }
        if (BAND && (hand_to == 4 || (SG_K0 && P.u_list && hand_to == 2 && nwin == 0))) {
            // the full-frame K1 after this kernel resumes the pair from its state: its
            // tail (§3.10), or all of it (K0: the first window already has D(0, 0) >
            // 30, an unrelated pair whose every window would go to a cooperative
            // warp, or is not band-shaped at all)
            list_push(P, false, pair);
            if (P.mixed) atomicSub(P.remaining, 1u);
            return;
        }
        if (BAND && hand_to == 2) atomicAdd(P.coop_out, 1u);  // before the pair is visible
        q_push(hand_to == 0 ? P.q_band : hand_to == 1 ? P.q_full : hand_to == 2 ? P.q_coop : P.q_std,
               P.n_pairs, pair);
    };

#ifdef SG_DEBUG_POST
    unsigned long long dbg_t0 = 0; int dbg_w0 = 0, dbg_t = 0, dbg_p = 0;
#endif
    auto finish_pair = [&]() {
#ifdef SG_DEBUG_POST
        if (!BAND && P.restore) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - dbg_t0 > 100000ull)
                printf("slow post pair %d: %llu ns, windows %d -> %d, n %d m %d, from toff %d poff %d dist %d status %x\n",
                       pair, t - dbg_t0, dbg_w0, nwin, n_tot, m_tot, dbg_t, dbg_p, dist, status);
        }
#endif
        if (cur_op >= 0) put_byte((static_cast<uint32_t>(cur_op) << 6) | (cur_len - 1));
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
            c[5] = static_cast<unsigned long long>(nwin) * static_cast<unsigned>(K + 1);
            c[6] = c_bequiv;
        }
        if (P.slice_done) {  // the pair's outputs are visible before its slice counts it
            __threadfence();
            atomicAdd(P.slice_done + pair / P.slice_pairs, 1u);
        }
        body_left(P, pair);
        if (P.mixed) atomicSub(P.remaining, 1u);
    };

    // Claim the next pair for the calling (possibly divergent) lanes.
    auto fetch = [&]() {
        pair = -1;
        bool restore = false;
        if (P.mixed) {  // a pair handed back by a cooperative warp first (if any is out)
            const bool back = !BAND || *reinterpret_cast<const volatile unsigned*>(P.coop_out) != 0u;
            pair = q_pop_warp(BAND ? P.q_band : P.q_full, P.n_pairs, back);
            if (BAND && pair >= 0) atomicSub(P.coop_out, 1u);
            restore = pair >= 0;
        }
        if (BAND || !P.mixed) {  // fresh pairs (warp-aggregated claim)
            const bool want = pair < 0 &&
                (!P.mixed || *reinterpret_cast<const volatile unsigned*>(P.next_pair) <
                                 static_cast<unsigned>(n_fresh));
            const unsigned active = __activemask();
            const unsigned wm = __ballot_sync(active, want);
            if (want) {
                const int leader = __ffs(wm) - 1;
                unsigned base = 0;
                if (lane == leader) base = atomicAdd(P.next_pair, static_cast<unsigned>(__popc(wm)));
                base = __shfl_sync(wm, base, leader);
                const int q = static_cast<int>(base + __popc(wm & ((1u << lane) - 1u)));
                pair = q < n_fresh ? (P.order ? P.order[q] : q) : -1;
                restore = P.restore != 0;
                if (P.warp_times && pair < 0 && ph_fresh_end == 0)  // diagnostics
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ph_fresh_end));
            }
        }
        if (pair < 0) return;
        n_tot = P.text_len[pair];
        m_tot = P.pat_len[pair];
        tbase = P.text_off[pair];
        pbase = P.pat_off[pair];
        {   // streamed upload: wait until the pair's sequence words have arrived
            const int64_t lw = (max(tbase + n_tot, pbase + m_tot) + 15) >> 4;
            const int64_t cw = lw / P.chunk_words;
            const int c = cw < P.n_chunks - 1 ? static_cast<int>(cw) : P.n_chunks - 1;
            while (*reinterpret_cast<const volatile unsigned*>(P.ready + c) == 0u) __nanosleep(1000);
        }
        hasn = P.has_n ? P.has_n[pair] != 0 : false;
        toff = poff = 0;
        dist = nwin = status = 0;
        window_cap = 4 * ((n_tot + m_tot) / step_limit + 2);  // aligner.cpp:40
        nx_tw = nx_pw = -1;
        outw = P.scratch + (P.bound_off[pair] >> 2);
        out_bytes = 0;
        cur_op = -1;
        cur_len = 0;
        acc = 0;
        acc_n = 0;
        c_stored = c_writes = c_reads = c_rows = c_cells = c_bequiv = 0;
        pass_win = 0;
#ifdef SG_DEBUG_POST
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dbg_t0));
#endif
        if (restore) {  // continue where the other frame stopped (state written before the push)
            const int4 rs = __ldcg(reinterpret_cast<const int4*>(P.resume_state + 4ll * pair));
            toff = rs.x;
            poff = rs.y;
            cur_op = (rs.z & 0xFF) == 0xFF ? -1 : (rs.z & 0xFF);
            cur_len = rs.z >> 8;
            acc = static_cast<uint32_t>(rs.w);
            dist = __ldcg(P.distance + pair);
            nwin = __ldcg(P.windows + pair);
#ifdef SG_DEBUG_POST
            dbg_w0 = nwin; dbg_t = toff; dbg_p = poff;
#endif
            out_bytes = __ldcg(P.out_bytes + pair);
            acc_n = out_bytes & 3;
            outw += out_bytes >> 2;
            if (P.counters) {
                const unsigned long long* c =
                    reinterpret_cast<const unsigned long long*>(P.counters + 7ll * pair);
                c_stored = __ldcg(c + 0);
                c_writes = __ldcg(c + 1);
                c_reads = __ldcg(c + 2);
                c_rows = __ldcg(c + 3);
                c_cells = __ldcg(c + 4);
                c_bequiv = __ldcg(c + 6);
            }
        }
    };

    // Matching bases from (i, j) on (0..16; 0 at a mismatch or a non-ACGT base).
    auto match_run = [&](int i, int j) -> int {
        const int bi = t_sh + i, bj = p_sh + j;
        const int si = 2 * (bi & 15), sj = 2 * (bj & 15);
        constexpr int RM = BAND ? 7 : 0xFFFF;  // band: ring slots
        const int wi = (tb0 + (bi >> 4)) & RM, wi1 = (tb0 + (bi >> 4) + 1) & RM;
        const int wj = (pb0 + (bj >> 4)) & RM, wj1 = (pb0 + (bj >> 4) + 1) & RM;
        const uint32_t t0 = lds_v(sq_t + wi * 32 + lane), t1 = lds_v(sq_t + wi1 * 32 + lane);
        const uint32_t p0 = lds_v(sq_p + wj * 32 + lane), p1 = lds_v(sq_p + wj1 * 32 + lane);
        uint32_t x = __funnelshift_r(t0, t1, si) ^ __funnelshift_r(p0, p1, sj);
        x = (x | (x >> 1)) & 0x55555555u;  // bit 2k: base k differs
        if (hasn) {
            const uint32_t tn = __funnelshift_r(sq_tn[(i >> 5) * 32 + lane],
                                                sq_tn[((i >> 5) + 1) * 32 + lane], i & 31);
            const uint32_t pn = __funnelshift_r(sq_pn[(j >> 5) * 32 + lane],
                                                sq_pn[((j >> 5) + 1) * 32 + lane], j & 31);
            uint32_t s = (tn | pn) & 0xFFFFu;  // bit k: base k is non-ACGT -> even bit 2k
            s = (s | (s << 8)) & 0x00FF00FFu;
            s = (s | (s << 4)) & 0x0F0F0F0Fu;
            s = (s | (s << 2)) & 0x33333333u;
            s = (s | (s << 1)) & 0x55555555u;
            x |= s;
        }
        return __clz(__brev(x)) >> 1;  // 16 when all 16 bases match
    };

    const long long dwarp = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (P.warp_times && lane == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.warp_times[dwarp * 3] = t;
    }
    unsigned long long last_busy = 0;
    bool need_pair = true, need_window = false, need_load = false;
    unsigned long long ph_setup = 0, ph_dc = 0, ph_tb = 0, ph_it = 0, ph_act = 0, ph_trips = 0,
                       ph_steps = 0, ph_tbn = 0, ph_idle = 0, ph_std = 0, ph_ffc = 0, ph_ffl = 0;
    for (;;) {
        const long long ck0 = clock64();
        // ---------------------------------------------- per-lane setup
        while (need_pair || need_window) {
            if (need_pair) {
                fetch();
                if (pair < 0) {
                    need_pair = P.mixed != 0;  // mixed: retry (work may be handed over)
                    break;
                }
                need_pair = false;
                need_window = true;
            }
            const int nw = status == 0 ? next_window() : 0;
            if (nw == 1) {
                need_load = true;
            } else if (nw == 2) {
                defer_pair();
                pair = -1;
                need_pair = true;
            } else {
                finish_pair();
                pair = -1;
                need_pair = true;
            }
            need_window = false;
        }
        if (need_load) {
            load_segment();
            need_load = false;
        }
        const bool in_dc = pair >= 0;
        if (!__any_sync(kFull, in_dc)) {
            if (!P.mixed || *reinterpret_cast<const volatile unsigned*>(P.remaining) == 0u) break;
            // a band warp with nothing left to take: no fresh pair, none out at a
            // cooperative warp (the only way one can come back)
            if (BAND && *reinterpret_cast<const volatile unsigned*>(P.next_pair) >=
                            static_cast<unsigned>(n_fresh) &&
                *reinterpret_cast<const volatile unsigned*>(P.coop_out) == 0u)
                break;

            // pairs are still in flight: one may be handed to this warp
            idle_wait(BAND ? 4000 : 16000);
            ph_idle += clock64() - ck0;
            continue;
        }
        __syncwarp();
        if (P.warp_times && lane == 0)  // diagnostics: the last iteration with work
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(last_busy));
        const long long ck1 = clock64();

        // ------------------------------------------------ DC chunks + d_opt detection
        // Up to kSubChunks chunks of R rows before the traceback phase, so
        // that more lanes reach it together; solved lanes sweep idle.
        bool solved = false;
        const int n_in = BAND ? 0 : __popc(__ballot_sync(kFull, in_dc));
        for (int sub = 0; sub < (BAND ? band_sub : kSubMax); ++sub) {
            const bool act = in_dc && !solved;
            if (BAND) {
                if (sub > 0 && !__any_sync(kFull, act)) break;
            } else if (sub > 0) {
                const int n_act = __popc(__ballot_sync(kFull, act));
                if (n_act == 0) break;
                if (sub >= kSubChunks && (n_in - n_act) * 32 >= n_in * kTbLanes) break;
            }
            if constexpr (BAND) {
                // (the main pass's band warps never hold an STD window: those are pair
                // tails, run by the tail K1 in the STD frame, §3.10)
                int fr = TAIL ? band_chunk<kBandR, true>(act, d0, W, cmax + 1, m_w, 0, bmem, two, hmul)
                              : band_chunk<kBandR, false>(act, d0, W, cmax + 1, K0, -e_lo, bmem, two, hmul);
                ++ph_it;
                ph_act += __popc(__ballot_sync(kFull, act));
                if (TAIL && act) {  // the STD frame is exact for every row
                    if (found_d < 0 && fr >= 0 && d0 + fr <= K) found_d = d0 + fr;
                    solved = found_d >= 0 || d0 + kBandR > K;
                    if (!solved) d0 += kBandR;
                } else if (act) {
                    if (found_d < 0 && fr >= 0) found_d = d0 + fr;
                    // D(0, 0) is exact up to band_last; beyond it the window goes
                    // to a cooperative warp
                    solved = found_d >= 0 || d0 + kBandR > band_last;
                    if (solved && (found_d < 0 || found_d > band_last)) {
                        defer_now = true;
                        hand_to = 2;
                    }
                    if (!solved) d0 += kBandR;
                }
                continue;
            }
            int fr = -1;
            if (!BAND && bnd_smem) {  // mixed full-frame warp: STD windows first
                // (compiled out: its traceback reads X / Y events, band_chunk writes planes)
                static_assert(band::FWARPS == 0, "band_chunk writes parity planes");
                const bool act_std = act && std_win;
                if (__any_sync(kFull, act_std)) {
                    const int f = band_chunk<4, true>(act_std, d0, W, C, m_w, 0, bmem, two, hmul);
                    if (act_std) fr = f;
                    ++ph_it;
                    ph_act += __popc(__ballot_sync(kFull, act_std));
                    ph_std += __popc(__ballot_sync(kFull, act_std));
                }
            }
            const bool act_full = act && !std_win;
            if (__any_sync(kFull, act_full)) {
                const int n_max = warp_max(act_full ? n_w : 0);
                const int f = dc_chunk<L, R, C>(act_full ? n_w : 0, act_full, m_w, act_full ? d0 : 0,
                                                n_max, two, one, lmem);
                if (act_full) fr = f;
                ph_ffc += 1;
                ph_ffl += __popc(__ballot_sync(kFull, act_full));
            }
            ++ph_it;
            ph_act += __popc(__ballot_sync(kFull, act));
            if (act) {
                if (found_d < 0 && fr >= 0 && d0 + fr <= K) found_d = d0 + fr;
                const bool seg_et = P.et || !first_seg;
                solved = seg_et ? (found_d >= 0 || d0 + R > K) : (d0 + R > K);
                if (!solved) d0 += R;
            }
        }
        __syncwarp();
        const long long ck2 = clock64();
        ph_setup += ck1 - ck0;
        ph_dc += ck2 - ck1;

        // ------------------------------------------------ TB + advance
        int tb_trip = 0;
        if (BAND && in_dc && solved && defer_now) {
            defer_now = false;
            defer_pair();
            pair = -1;
            need_pair = true;
        } else if (in_dc && solved) {
            // single window with D(0, 0) > k: not found (batch.cpp:57-62)
            const bool not_found = P.single && found_d < 0;
            if (found_d < 0 && !not_found) status = kStInternal | kDetNoStep;  // aligner.cpp:69-70
            if (first_seg) {
                last_d = found_d;
                // reference counters for this logical window (dp.cpp:23-37,58-75,225-228)
                const int rows_ref = P.et && found_d >= 0 ? found_d + 1 : K + 1;
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
                c_bequiv += 3ull * (n_w + 1) * static_cast<unsigned long long>(K + 1) * m_w;
            } else if (found_d != expect_d) {
                status = kStInternal | kDetSegment;
            }
            if (not_found) {
                dist = -1;
                ++nwin;
                ++pass_win;
                toff = n_tot;
                poff = m_tot;
                need_window = true;
            } else {
            // GenASM-TB (traceback.cpp:56-113). On the path D(i,j) == d, so
            // Match <=> t_i == p_j (both ACGT) and runs of matches are taken
            // at once; at a mismatch the events pick Sub > Del > Ins.
            const int off = WB - m_w;
            int i = 0, j = 0, d = found_d < 0 ? 0 : found_d, steps = 0;
            const int lim = limit >= 0 ? limit : 0x3FFFFFFF;
            unsigned reads = 0;
            ++ph_tbn;
            // interior: both sides left, inside the stored event columns. One
            // trip takes a run of matches and then, where the run stopped at a
            // mismatch, the edit there (its event words load after the run).
            auto emit_short = [&](int op, int k) {  // k <= 16: extend the open byte or write it
                if (op == cur_op && cur_len + k <= 64) {
                    cur_len += k;
                } else {
                    const bool same = op == cur_op;
                    const uint32_t byte = (static_cast<uint32_t>(cur_op) << 6) |
                                          static_cast<uint32_t>(same ? 63 : cur_len - 1);
                    if (cur_op >= 0) put_byte(byte);
                    cur_len = same ? cur_len + k - 64 : k;
                    cur_op = op;
                }
            };
            if constexpr (BAND) {
                // band windows: n_w = W > lim = cmax, so the walk stops at the step
                // limit or at the end of the pattern (m_w >= W - 30; the tail below
                // takes the deletions left)
                const int dm = d0 + kBandR - 1;  // the window's last computed row
                // the bit of (i + 1, j + 1): band j - i - e_lo, STD (tail K1) j + 1
                int kb = TAIL ? 1 : -e_lo;
                // table reads (dp.hpp:46-66): 3 per step while d > 0, 1 after; s0 =
                // the step count when d reached 0
                int s0 = d == 0 ? 0 : -1;
                while (steps < lim && j < m_w) {
                    ++ph_steps;
                    ++tb_trip;
                    const int run = match_run(i, j);
                    const int k = min(run, min(lim - steps, m_w - j));
                    i += k;
                    j += k;
                    steps += k;
                    if (k > 0) emit_short(0, k);
                    if (k != run || run == 16 || steps == lim || j == m_w) continue;
                    // the edit at the mismatch (i, j), from the parity planes of column
                    // i + 1 (§3.8): a cell held by n of rows 0..dm has D = dm + 1 - n;
                    // P0 = n & 1, P1 = (odd rows holding it) & 1. The two neighbours of a
                    // path cell are within 1 of d, so D(nbr) == d - 1 <=> (P0, P1) ==
                    // (E0, E1). (i + 1, j + 1) is at bit kb, (i + 1, j) at kb - 1.
                    if (TAIL) kb = j + 1;  // (the STD frame: bit j + 1)
                    if (static_cast<unsigned>(kb) >= 32u) {  // cannot happen for d <= 30
                        status = kStInternal | kDetSegment;
                        break;
                    }
                    const uint2 pl = *reinterpret_cast<const uint2*>(xy + (i + 1) * 64 + lane * 2);
                    const uint32_t e0 = static_cast<uint32_t>(dm - d) & 1u;
                    const uint32_t e1 = static_cast<uint32_t>(((dm + 1) >> 1) - ((d - 1) >> 1)) & 1u;
                    const uint32_t lt = (pl.x ^ (e0 - 1u)) & (pl.y ^ (e1 - 1u));  // D(nbr) == d - 1
                    const int op = (lt >> kb) & 1u ? 1 : (((lt << 1) >> kb) & 1u ? 3 : 2);
                    if (d == 0) status = kStInternal | kDetNoStep;
                    i += op != 2;
                    j += op != 3;
                    kb += (op == 2) - (op == 3);
                    --d;
                    ++dist;
                    ++steps;
                    if (d == 0) s0 = steps;
                    emit_short(op, 1);
                }
                if (s0 < 0) s0 = steps;
                reads += 2u * static_cast<unsigned>(s0) + static_cast<unsigned>(steps);
            } else
            for (;;) {
                ++ph_steps;
                ++tb_trip;
                int rem = lim - steps;
                if (rem == 0 || i == n_w || j == m_w || i >= cmax) break;
                const int run = match_run(i, j);
                const int k = min(min(run, rem), min(min(n_w - i, m_w - j), cmax - i));
                if (k > 0) {
                    reads += static_cast<unsigned>(k) * (d == 0 ? 1u : 3u);
                    i += k;
                    j += k;
                    steps += k;
                    rem -= k;
                    emit_short(0, k);
                }
                if (k != run || run == 16 || rem == 0 || i == n_w || j == m_w || i >= cmax) continue;
                // the edit at the mismatch (i, j)
                int op;
                if constexpr (BAND) {
                    // parity planes of column i + 1 (§3.8): a cell with n = #(rows
                    // 0..dm holding it) has D = dm + 1 - n; P0 = n & 1, P1 = #(odd
                    // rows holding it) & 1. The two neighbours of a path cell are
                    // within 1 of d, so D(nbr) == d - 1 <=> (P0, P1) == (E0, E1).
                    const uint2 pl = *reinterpret_cast<const uint2*>(xy + (i + 1) * 64 + lane * 2);
                    const int dm = d0 + kBandR - 1;  // the window's last computed row
                    const uint32_t e0 = static_cast<uint32_t>(dm - d) & 1u;
                    const uint32_t e1 = static_cast<uint32_t>(((dm + 1) >> 1) - ((d - 1) >> 1)) & 1u;
                    const uint32_t lt = (pl.x ^ (e0 - 1u)) & (pl.y ^ (e1 - 1u));  // D(nbr) == d - 1
                    int kb;  // the bit of (i + 1, j + 1); (i + 1, j) is the one below
                    if (std_win) {
                        kb = j + 1;
                    } else {  // diagonal band: cell (i, j) at bit j - i - e_lo
                        kb = j - i - e_lo;
                        if (static_cast<unsigned>(kb) >= 32u) {  // cannot happen for d <= 30
                            status = kStInternal | kDetSegment;
                            break;
                        }
                    }
                    op = (lt >> kb) & 1u ? 1 : (((lt << 1) >> kb) & 1u ? 3 : 2);
                } else {
                    const uint2 ev = *reinterpret_cast<const uint2*>(xy + i * 64 + lane * 2);
                    uint32_t bit;
                    const unsigned q = static_cast<unsigned>(j + off);
                    const int dp = static_cast<int>(q / L) - band_base<L>(i, off);
                    if (!std_win && static_cast<unsigned>(dp) >= 32u / L) break;  // left the band
                    bit = std_win ? 1u << j : 0x80000000u >> ((32 / L) * (q % L) + dp);
                    op = ev.x & bit ? 1 : (ev.y & bit ? 3 : 2);
                }
                if (d == 0) status = kStInternal | kDetNoStep;
                reads += d == 0 ? 1u : 3u;
                i += op != 2;
                j += op != 3;
                --d;
                ++dist;
                ++steps;
                emit_short(op, 1);
            }
            // tail: one side consumed (a single run of indels), or the next
            // column has no stored events (continue on the suffix)
            bool cont = false;
            {
                const int rem = lim - steps;
                if (rem > 0 && !(i == n_w && j == m_w)) {
                    if (i == n_w || j == m_w) {
                        const int op = i == n_w ? 2 : 3;
                        const int left = i == n_w ? m_w - j : n_w - i;
                        if (d != left)
                            status = kStInternal | (i == n_w ? kDetBudgetI : kDetBudgetD);
                        const int k = min(rem, left);
                        i += op != 2 ? k : 0;
                        j += op != 3 ? k : 0;
                        d -= k;
                        dist += k;
                        steps += k;
                        emit(op, k);
                    } else {
                        cont = true;
                    }
                }
            }
            if (!P.single) c_reads += reads;  // single window: counted before TB (aligner.cpp:98-99)
            if (BAND && cont) status = kStInternal | kDetSegment;  // non-final: W - O <= cmax
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
                need_load = true;
            } else {
                if (!cont && limit < 0 && d != 0) status = kStInternal | kDetLeftover;
                toff += i;
                poff += j;
                ++nwin;
                ++pass_win;
                if (nwin > window_cap) status = kStInternal | kDetWatchdog;
                need_window = true;
            }
            }  // found
        }
        __syncwarp();
        ph_tb += clock64() - ck2;
        if (P.phase_cycles) ph_trips += warp_max(tb_trip);
    }
    if (P.warp_times && lane == 0) {  // diagnostics: when each warp leaves, on which SM
        unsigned long long t, smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(*reinterpret_cast<unsigned*>(&smid)));
        P.warp_times[dwarp * 3 + 1] = last_busy ? last_busy : t;
        P.warp_times[dwarp * 3 + 2] = __reduce_max_sync(kFull, static_cast<unsigned>(ph_fresh_end >> 20)) ;
    }
    if (P.phase_cycles) {
        ph_steps = __reduce_add_sync(kFull, static_cast<unsigned>(ph_steps));
        ph_tbn = __reduce_add_sync(kFull, static_cast<unsigned>(ph_tbn));
        if (lane == 0) {  // band warps [0, 9), full-frame warps [9, 18)
            unsigned long long* pc = P.phase_cycles + (BAND ? 0 : 9);
            atomicAdd(pc + 0, ph_setup);
            atomicAdd(pc + 1, ph_dc);
            atomicAdd(pc + 2, ph_tb);
            atomicAdd(pc + 3, ph_it);
            atomicAdd(pc + 4, ph_act);
            atomicAdd(pc + 5, ph_trips);
            atomicAdd(pc + 6, ph_steps);
            atomicAdd(pc + 7, ph_tbn);
            atomicAdd(pc + 8, ph_idle);
            if (!BAND) {
                atomicAdd(P.phase_cycles + 18, ph_std);
                atomicAdd(P.phase_cycles + 19, ph_ffc);
                atomicAdd(P.phase_cycles + 20, ph_ffl);
            }
        }
    }
}

// ------------------------------------------------------ K1c: cooperative windows
//
// DESIGN.md §3.9. One warp computes one window of W <= 64 columns: the standard
// frame with 64-bit rows (bit j = cell (i, j), complemented: 1 <=> D(i, j) <= d),
// lane r computes row 32p + r of pass p, one column per step, one column behind
// lane r - 1 (its north neighbour arrives by shuffle; lane 0 reads the previous
// pass's last row). Cell update (dp.cpp:187-211 in these coordinates):
//   C[i][d] = (sh(C[i+1][d]) & EQ_i) | C[i+1][d-1] | sh(C[i+1][d-1]) | sh(C[i][d-1])
// with sh(x) = x >> 1 and, when m_w = 64, the end-of-pattern cell D(i', 64) =
// n_w - i' shifted in at bit 63 (dp.hpp:145-154). Traceback events X / Y of
// every row are OR-ed into shared memory (atom.shared.or.b64), so the traceback
// is K1's. Used for the full-width windows the single-word frames cannot take
// (D(0, 0) > 30, or 32 <= m_w with |m_w - n_w| > 30): 30..60 rows in one or
// two passes instead of 8..16 sequential 4-row chunks on one lane.
namespace coop {
constexpr int kWords = 66 * 2 + 66 * 2 + 65 * 4 + 20 + 8;  // eq, prow, xy (+ dummies), staging, held pairs
}

__device__ __forceinline__ uint64_t shr1_in(uint64_t x, uint32_t b) {
    return (x >> 1) | (static_cast<uint64_t>(b) << 63);
}

// init column (i = n_w) of row d: bits j in [m - d, m] (bit 64 = the boundary, implicit)
__device__ __forceinline__ uint64_t coop_init(int d, int m) {
    if (d < 0) return 0ull;
    const int lo = max(m - d, 0);
    const uint64_t top = m >= 63 ? ~0ull : ((2ull << m) - 1ull);
    return lo >= 64 ? 0ull : (top & (~0ull << lo));
}

__device__ void coop_body(const AlignParams& P, uint32_t* const sm) {
    const int lane = threadIdx.x & 31;
    uint2* const eqs = reinterpret_cast<uint2*>(sm);             // [64 + dummy] EQ_i
    uint2* const prow = eqs + 66;                                // [64 + 2 dummies] last row of the pass
    uint4* const xys = reinterpret_cast<uint4*>(prow + 66);      // [64 + dummy] X lo, X hi, Y lo, Y hi
    uint32_t* const st = reinterpret_cast<uint32_t*>(xys + 65);  // text [6], pattern [6], tn [3], pn [3]
    const int W = P.W, step_limit = W - P.O, K = W;
    const long long dwarp = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (P.warp_times && lane == 0) {  // diagnostics: start, last window's end
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.warp_times[dwarp * 3] = t;
        P.warp_times[dwarp * 3 + 1] = t;
    }
    // lane 0: pairs taken in one pop (in shared memory: as a local array they were the
    // kernel's only stack frame)
    int* const held = reinterpret_cast<int*>(st + 20);
    int nheld = 0, next_held = 0;
    for (;;) {
        int pair = -1;
        if (lane == 0) {
            if (next_held == nheld) {
                next_held = 0;
                nheld = q_pop_n(P.q_coop, P.n_pairs, 8, held);
            }
            if (next_held < nheld) pair = held[next_held++];
        }
        pair = __shfl_sync(kFull, pair, 0);
        if (pair < 0) {
            if (*reinterpret_cast<const volatile unsigned*>(P.remaining) == 0u) break;
            idle_wait(2 * band::kCoopSleep);  // ~ns at 2 GHz
            continue;
        }
        // ---- restore the pair (every lane holds the same state; lane 0 writes)
        const int n_tot = P.text_len[pair], m_tot = P.pat_len[pair];
        const int64_t tbase = P.text_off[pair], pbase = P.pat_off[pair];
        const bool hasn = P.has_n ? P.has_n[pair] != 0 : false;
        const int4 rs = __ldcg(reinterpret_cast<const int4*>(P.resume_state + 4ll * pair));
        int toff = rs.x, poff = rs.y;
        int cur_op = (rs.z & 0xFF) == 0xFF ? -1 : (rs.z & 0xFF), cur_len = rs.z >> 8;
        uint32_t acc = static_cast<uint32_t>(rs.w);
        int dist = __ldcg(P.distance + pair), nwin = __ldcg(P.windows + pair);
        int out_bytes = __ldcg(P.out_bytes + pair), acc_n = out_bytes & 3, status = 0;
        uint32_t* outw = P.scratch + (P.bound_off[pair] >> 2) + (out_bytes >> 2);
        unsigned long long cn[7] = {0, 0, 0, 0, 0, 0, 0};
        if (P.counters) {
            const unsigned long long* c =
                reinterpret_cast<const unsigned long long*>(P.counters + 7ll * pair);
#pragma unroll
            for (int k = 0; k < 7; ++k) cn[k] = __ldcg(c + k);
        }
        const int window_cap = 4 * ((n_tot + m_tot) / step_limit + 2);  // aligner.cpp:40
        auto put_byte = [&](uint32_t b) {
            acc |= b << (8 * acc_n);
            ++out_bytes;
            if (++acc_n == 4) {
                if (lane == 0) *outw = acc;
                ++outw;
                acc = 0;
                acc_n = 0;
            }
        };
        auto emit = [&](int op, int len) {  // cigar_append (cigar.cpp:9-16) as run bytes
            if (op == cur_op && cur_len + len <= 64) {
                cur_len += len;
                return;
            }
            if (op == cur_op) {
                len -= 64 - cur_len;
                cur_len = 64;
            }
            if (cur_op >= 0) put_byte((static_cast<uint32_t>(cur_op) << 6) | (cur_len - 1));
            while (len > 64) {
                put_byte((static_cast<uint32_t>(op) << 6) | 63u);
                len -= 64;
            }
            cur_op = op;
            cur_len = len;
        };
        int hand = -1;  // -1 finished, 0 band, 1 full frame
        int last_d = 0, pass_win = 0;
        for (;;) {
            // ---- next window (aligner.cpp:44-64)
            const int n_rem = n_tot - toff, m_rem = m_tot - poff;
            if (n_rem == 0 || m_rem == 0) {
                if (n_rem + m_rem > 0) {  // aligner.cpp:48-57
                    emit(n_rem == 0 ? 2 : 3, n_rem + m_rem);
                    dist += n_rem + m_rem;
                }
                break;
            }
            const bool fin = n_rem <= W && m_rem <= W;
            const int n_w = min(W, n_rem), m_w = min(W, m_rem), dl = m_w - n_w;
            const bool band_ok = !fin && n_w == W && dl <= band::kLastRow && dl >= -band::kLastRow;
            if (pass_win > 0 && band_ok && last_d <= band::kBackRow) { hand = 0; break; }
            // an STD window (m_w <= 31): the pair's tail, for the tail K1 (§3.10)
            if (P.t_list && !fin && n_w == W && m_w <= 31) { hand = 5; break; }
            // this warp takes every other window: final ones (traceback to the
            // end, events of every column) and the tails of the STD queue too
            const int lim = fin ? 0x3FFFFFFF : step_limit, cap = fin ? n_w : step_limit;
            const long long cw0 = clock64();
            // ---- staging: the window's packed text / pattern (bases 16k.. in word k) and N bits
            {
                const int64_t ta = tbase + toff, pa = pbase + poff;
                const uint32_t rt = lane < 7 ? __ldcg(P.seq + (ta >> 4) + lane) : 0u;
                const uint32_t rp = lane < 7 ? __ldcg(P.seq + (pa >> 4) + lane) : 0u;
                const uint32_t rt1 = __shfl_down_sync(kFull, rt, 1), rp1 = __shfl_down_sync(kFull, rp, 1);
                if (lane < 6) {
                    st[lane] = __funnelshift_r(rt, rt1, 2 * static_cast<int>(ta & 15));
                    st[6 + lane] = __funnelshift_r(rp, rp1, 2 * static_cast<int>(pa & 15));
                }
                uint32_t tn = 0, pn = 0;
                if (hasn) {
                    const int64_t a = lane < 3 ? ta : pa;
                    const int k = lane < 3 ? lane : lane - 3;
                    const uint32_t r0 = lane < 6 ? __ldcg(P.nmask + (a >> 5) + k) : 0u;
                    const uint32_t r1 = lane < 6 ? __ldcg(P.nmask + (a >> 5) + k + 1) : 0u;
                    const uint32_t w = __funnelshift_r(r0, r1, static_cast<int>(a & 31));
                    if (lane < 3) tn = w; else pn = w;
                }
                if (lane < 3) st[12 + lane] = tn;
                else if (lane < 6) st[15 + lane - 3] = pn;
                // events start empty; column lane and lane + 32
                xys[lane] = make_uint4(0u, 0u, 0u, 0u);
                xys[lane + 32] = make_uint4(0u, 0u, 0u, 0u);
            }
            __syncwarp();
            // pattern code planes (64 bits, j < m_w, no N) and EQ_i of columns lane, lane + 32
            {
                uint64_t lo = 0, hi = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t w = st[6 + k];
                    lo |= static_cast<uint64_t>(compress_stride<2>(w & 0x55555555u)) << (16 * k);
                    hi |= static_cast<uint64_t>(compress_stride<2>((w >> 1) & 0x55555555u)) << (16 * k);
                }
                uint64_t valid = m_w >= 64 ? ~0ull : ((1ull << m_w) - 1ull);
                if (hasn) valid &= ~(static_cast<uint64_t>(st[15]) | (static_cast<uint64_t>(st[16]) << 32));
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int i = lane + 32 * h;
                    const int code = static_cast<int>((st[i >> 4] >> (2 * (i & 15))) & 3u);
                    const uint64_t l = code & 1 ? lo : ~lo, g = code & 2 ? hi : ~hi;
                    uint64_t e = l & g & valid;
                    if (hasn && ((st[12 + (i >> 5)] >> (i & 31)) & 1u)) e = 0ull;
                    eqs[i] = make_uint2(static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32));
                }
            }
            __syncwarp();
            // ---- DC: passes of 32 rows
            int found = -1;
            for (int p = 0; 32 * p <= K && found < 0; ++p) {
                const int d = 32 * p + lane;
                uint64_t v = coop_init(d, m_w), dg = coop_init(d - 1, m_w);
                bool f0 = false;
                // branch-free steps: inactive lanes (not started / finished) keep
                // their state; their event and row stores go to the dummy slots
                const uint64_t pmask = p > 0 ? ~0ull : 0ull;
                for (int s = 0; s < n_w + 31; ++s) {
                    const uint32_t ul = __shfl_up_sync(kFull, static_cast<uint32_t>(v), 1);
                    const uint32_t uh = __shfl_up_sync(kFull, static_cast<uint32_t>(v >> 32), 1);
                    const int col = n_w - 1 - s + lane;
                    const bool act = lane <= s && col >= 0;
                    const int cs = act ? col : 64;  // column slot (64 = dummy)
                    const uint2 pr = prow[cs];
                    const uint2 e2 = eqs[cs];
                    uint64_t north = (static_cast<uint64_t>(uh) << 32) | ul;
                    if (lane == 0) north = ((static_cast<uint64_t>(pr.y) << 32) | pr.x) & pmask;
                    const uint64_t eq = (static_cast<uint64_t>(e2.y) << 32) | e2.x;
                    uint32_t be = 0, bs = 0, bn = 0;
                    if (m_w == 64) {  // D(i', 64) = n_w - i' <= d' shifted in at bit 63
                        const int c = n_w - col;
                        be = c - 1 <= d;
                        bs = c - 1 <= d - 1;
                        bn = c <= d - 1;
                    }
                    const uint64_t mt = shr1_in(v, be);
                    const uint64_t nc = (mt & eq) | dg | shr1_in(dg, bs) | shr1_in(north, bn);
                    {   // events: at one step the lanes are on different columns and lane
                        // r + 1 reaches a column one step after lane r, so the
                        // read-modify-write is race-free
                        const uint64_t x = mt & ~nc, y = v & ~nc;
                        const int es = act && col < cap ? col : 64;
                        uint4 o = xys[es];
                        o.x |= static_cast<uint32_t>(x);
                        o.y |= static_cast<uint32_t>(x >> 32);
                        o.z |= static_cast<uint32_t>(y);
                        o.w |= static_cast<uint32_t>(y >> 32);
                        xys[es] = o;
                    }
                    prow[lane == 31 ? cs : 65] = make_uint2(static_cast<uint32_t>(nc),
                                                            static_cast<uint32_t>(nc >> 32));
                    f0 |= act && col == 0 && (nc & 1ull);
                    dg = act ? north : dg;
                    v = act ? nc : v;
                }
                const unsigned fb = __ballot_sync(kFull, f0 && d <= K);
                if (fb) found = 32 * p + __ffs(fb) - 1;
                __syncwarp();
            }
            const long long cw1 = clock64();
            if (found < 0) {  // D(0, 0) > K (aligner.cpp:69-70)
                status = kStInternal | kDetNoStep;
                break;
            }
            // reference counters of the window (dp.cpp:23-37,58-75,225-228)
            {
                const int rows_ref = P.et ? found + 1 : K + 1;
                int pol = P.policy;
                if (fin && pol == 2) pol = 1;  // final window: DENT -> SENE (aligner.cpp:79)
                int keep_cols = n_w + 1, keep_bits = m_w;
                if (pol == 2) {
                    keep_cols = min(n_w, step_limit) + 1;
                    keep_bits = min(m_w, step_limit + 1);
                }
                const unsigned long long slots = pol == 0 ? 3ull : 1ull;
                cn[0] += static_cast<unsigned long long>(rows_ref) * keep_cols * keep_bits * slots;
                cn[1] += static_cast<unsigned long long>(rows_ref) * keep_cols * slots;
                cn[3] += rows_ref;
                cn[4] += static_cast<unsigned long long>(rows_ref) * n_w;
                cn[6] += 3ull * (n_w + 1) * static_cast<unsigned long long>(K + 1) * m_w;
            }
            // ---- TB (traceback.cpp:56-113), uniform over the lanes
            int i = 0, j = 0, d = found, steps = 0;
            unsigned reads = 0;
            for (;;) {
                int rem = lim - steps;
                if (rem == 0 || i == n_w || j == m_w) break;
                int run;
                {   // matching bases from (i, j) on
                    const uint32_t tw = __funnelshift_r(st[i >> 4], st[(i >> 4) + 1], 2 * (i & 15));
                    const uint32_t pw = __funnelshift_r(st[6 + (j >> 4)], st[6 + (j >> 4) + 1], 2 * (j & 15));
                    uint32_t x = tw ^ pw;
                    x = (x | (x >> 1)) & 0x55555555u;
                    if (hasn) {
                        const uint32_t tn = __funnelshift_r(st[12 + (i >> 5)], st[13 + (i >> 5)], i & 31);
                        const uint32_t pn = __funnelshift_r(st[15 + (j >> 5)], st[16 + (j >> 5)], j & 31);
                        uint32_t q = (tn | pn) & 0xFFFFu;
                        q = (q | (q << 8)) & 0x00FF00FFu;
                        q = (q | (q << 4)) & 0x0F0F0F0Fu;
                        q = (q | (q << 2)) & 0x33333333u;
                        q = (q | (q << 1)) & 0x55555555u;
                        x |= q;
                    }
                    run = __clz(__brev(x)) >> 1;
                }
                const int k = min(min(run, rem), min(n_w - i, m_w - j));
                if (k > 0) {
                    reads += static_cast<unsigned>(k) * (d == 0 ? 1u : 3u);
                    i += k;
                    j += k;
                    steps += k;
                    rem -= k;
                    emit(0, k);
                }
                if (k != run || run == 16 || rem == 0 || i == n_w || j == m_w) continue;
                const uint4 ev = xys[i];
                const uint32_t xw = j < 32 ? ev.x : ev.y, yw = j < 32 ? ev.z : ev.w;
                const int op = (xw >> (j & 31)) & 1u ? 1 : ((yw >> (j & 31)) & 1u ? 3 : 2);
                if (d == 0) status = kStInternal | kDetNoStep;
                reads += d == 0 ? 1u : 3u;
                i += op != 2;
                j += op != 3;
                --d;
                ++dist;
                ++steps;
                emit(op, 1);
            }
            {   // one side consumed: a single run of indels (traceback.cpp:76-86)
                const int rem = lim - steps;
                if (rem > 0 && !(i == n_w && j == m_w) && (i == n_w || j == m_w)) {
                    const int op = i == n_w ? 2 : 3;
                    const int left = i == n_w ? m_w - j : n_w - i;
                    if (d != left) status = kStInternal | (i == n_w ? kDetBudgetI : kDetBudgetD);
                    const int k = min(rem, left);
                    i += op != 2 ? k : 0;
                    j += op != 3 ? k : 0;
                    d -= k;
                    dist += k;
                    emit(op, k);
                }
            }
            if (fin && d != 0 && status == 0) status = kStInternal | kDetLeftover;  // traceback.cpp:110-111
            cn[2] += reads;
            toff += i;
            poff += j;
            ++nwin;
            ++pass_win;
            last_d = found;
            if (P.warp_times && lane == 0) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                P.warp_times[dwarp * 3 + 1] = t;
            }
            if (P.phase_cycles && lane == 0) {
                atomicAdd(P.phase_cycles + 21, 1ull);
                atomicAdd(P.phase_cycles + 22, static_cast<unsigned long long>(cw1 - cw0));
                atomicAdd(P.phase_cycles + 23, static_cast<unsigned long long>(clock64() - cw1));
                atomicAdd(P.phase_cycles + 24, static_cast<unsigned long long>(found));
            }
            if (nwin > window_cap) status = kStInternal | kDetWatchdog;
            if (status) break;
            __syncwarp();
        }
        // ---- finish the pair or hand it on
        if (lane == 0) {
            if (hand < 0) {
                if (cur_op >= 0) {
                    acc |= ((static_cast<uint32_t>(cur_op) << 6) | (cur_len - 1)) << (8 * acc_n);
                    ++out_bytes;
                    *outw = acc;
                } else if (acc_n) {
                    *outw = acc;
                }
                P.distance[pair] = dist;
                P.windows[pair] = nwin;
                P.status[pair] = status;
                P.out_bytes[pair] = out_bytes;
                if (P.counters) {
                    uint64_t* c = P.counters + 7ll * pair;
#pragma unroll
                    for (int k = 0; k < 7; ++k) c[k] = cn[k];
                    c[5] = static_cast<unsigned long long>(nwin) * static_cast<unsigned>(K + 1);
                }
                if (P.slice_done) {
                    __threadfence();
                    atomicAdd(P.slice_done + pair / P.slice_pairs, 1u);
                }
                body_left(P, pair);
                atomicSub(P.remaining, 1u);
                atomicSub(P.coop_out, 1u);
            } else {
                P.distance[pair] = dist;
                P.windows[pair] = nwin;
                P.status[pair] = 0;
                P.out_bytes[pair] = out_bytes;
                if (P.counters) {
                    uint64_t* c = P.counters + 7ll * pair;
#pragma unroll
                    for (int k = 0; k < 7; ++k) c[k] = cn[k];
                }
                int32_t* r = P.resume_state + 4ll * pair;
                r[0] = toff;
                r[1] = poff;
                r[2] = (cur_op & 0xFF) | (cur_len << 8);
                r[3] = static_cast<int32_t>(acc);
                if (hand == 5) {
                    list_push(P, true, pair);
                    atomicSub(P.remaining, 1u);
                    atomicSub(P.coop_out, 1u);
                } else {
                    q_push(hand == 0 ? P.q_band : hand == 1 ? P.q_full : P.q_std, P.n_pairs, pair);
                }
            }
        }
        __syncwarp();
    }
}

template <int L>
__global__ void __launch_bounds__(32 * KCfg<L>::WARPS, KCfg<L>::MINB)
    k1_window_align(const __grid_constant__ AlignParams P) {
    extern __shared__ uint32_t smem[];
    const int wib = threadIdx.x >> 5;
    k1_body<L, false>(P, smem + wib * warp_smem_words<L>(),
                      static_cast<long long>(blockIdx.x) * KCfg<L>::WARPS + wib, nullptr, nullptr);
}

// K1 mixed (§3.8): band warps (K1b) and full-frame warps (limb count LF) in one
// persistent block per SM, handing pairs to each other through P.q_full / P.q_band.
// A full-frame warp of the mixed kernel: K1<LF> memory, its parked rows
// [32 LF + 5][32][LF] and the STD windows' (EQ, parked) [68][32] uint2 — the same
// words as the parked rows for LF = 2 (same per-lane mapping), after them for LF = 1.
template <int LF> __host__ __device__ constexpr int mixed_eqp_offset() {
    return LF == 2 ? 0 : (32 * LF + 5) * 32 * LF;
}
template <int LF> __host__ __device__ constexpr int mixed_full_words() {
    return warp_smem_words<LF>() +
           ((32 * LF + 5) * 32 * LF > mixed_eqp_offset<LF>() + band::eqp_words()
                ? (32 * LF + 5) * 32 * LF : mixed_eqp_offset<LF>() + band::eqp_words());
}
template <int LF> __host__ __device__ constexpr int mixed_block_words() {
    return band::WARPS * k1_warp_words<2, true>() + band::FWARPS * mixed_full_words<LF>() +
           band::CWARPS * coop::kWords;
}
constexpr int kMixedWarps = band::WARPS + band::FWARPS + band::CWARPS;
template <int LF>
__global__ void __launch_bounds__(32 * kMixedWarps, 1)
    k1_mixed(const __grid_constant__ AlignParams P) {
    extern __shared__ uint32_t smem[];
    const int wib = threadIdx.x >> 5;
    if (wib >= band::WARPS + band::FWARPS) {
        coop_body(P, smem + band::WARPS * k1_warp_words<2, true>() +
                         band::FWARPS * mixed_full_words<LF>() +
                         (wib - band::WARPS - band::FWARPS) * coop::kWords);
    } else if (wib < band::WARPS) {
        if (wib * static_cast<int>(gridDim.x) + static_cast<int>(blockIdx.x) >= P.band_active)
            return;  // whole-rounds sizing: fewer band warps than slots, spread over the SMs
        k1_body<2, true>(P, smem + wib * k1_warp_words<2, true>(),
                         static_cast<long long>(blockIdx.x) * band::WARPS + wib, nullptr, nullptr);
    } else if constexpr (band::FWARPS > 0) {
        const int fw = wib - band::WARPS;
        uint32_t* const base = smem + band::WARPS * k1_warp_words<2, true>() + fw * mixed_full_words<LF>();
        k1_body<LF, false>(P, base, static_cast<long long>(blockIdx.x) * band::FWARPS + fw,
                           base + warp_smem_words<LF>(),
                           base + warp_smem_words<LF>() + mixed_eqp_offset<LF>());
    }
}

// The tail K1 (§3.10): the band warps alone (no cooperative warp), running the STD
// windows of the pairs the mixed kernel left in its tail list.
__global__ void __launch_bounds__(32 * band::WARPS, 1) k1_tail(const __grid_constant__ AlignParams P) {
    extern __shared__ uint32_t smem[];
    const int wib = threadIdx.x >> 5;
    if (P.wait_count) {
        // pipelined launch (§3.12): this slice's pairs are still leaving K1 mixed, which
        // runs beside this kernel on the other SMs and never waits for it. The wait is
        // bounded: a count that stays short is an internal error, not a hang.
        if (threadIdx.x == 0) {
            unsigned long long t0, t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            while (*reinterpret_cast<const volatile unsigned*>(P.wait_count) < P.wait_target) {
                __nanosleep(2000);
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t - t0 > 60000000000ull) {  // 60 s
                    atomicExch(P.pipe_err, 1u);
                    break;
                }
            }
            __threadfence();
        }
        __syncthreads();
    }
    k1_body<2, true, true>(P, smem + wib * k1_warp_words<2, true>(),
                           static_cast<long long>(blockIdx.x) * band::WARPS + wib, nullptr, nullptr);
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

template <int LF> int launch_mixed_L(const AlignParams& p, int grid, void* stream) {
    const size_t smem = static_cast<size_t>(mixed_block_words<LF>()) * 4;
    cudaError_t e = cudaFuncSetAttribute(k1_mixed<LF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
    k1_mixed<LF><<<grid, 32 * kMixedWarps, smem,
                   static_cast<cudaStream_t>(stream)>>>(p);
    return static_cast<int>(cudaGetLastError());
}

__global__ void k1_queue_init(uint32_t* q_band, uint32_t* q_full, uint32_t* q_coop,
                              uint32_t* q_std, unsigned* remaining, int n, const int32_t* n_dev) {
    if (n_dev) n = *n_dev;
    if (threadIdx.x < 32) {
        q_band[threadIdx.x] = 0u;
        q_full[threadIdx.x] = 0u;
        q_coop[threadIdx.x] = 0u;
        q_std[threadIdx.x] = 0u;
    }
    if (threadIdx.x == 0) *remaining = static_cast<unsigned>(n);
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

constexpr int kSliceBlock = 256;  // small: co-resident with K1's persistent blocks

__global__ void __launch_bounds__(kSliceBlock)
    k2_slice_scan(const int32_t* __restrict__ bytes, int64_t* __restrict__ dense_off, int32_t lo,
                  int32_t hi, const unsigned* __restrict__ slice_done, int s, int64_t* info) {
    __shared__ long long warp_tot[kSliceBlock / 32];
    __shared__ long long carry;
    if (threadIdx.x == 0) {
        const unsigned want = static_cast<unsigned>(hi - lo);
        // (null: the launches before this one on the stream finished the slice, §3.12)
        while (slice_done && *reinterpret_cast<const volatile unsigned*>(slice_done + s) < want)
            __nanosleep(2000);
        __threadfence();
        carry = lo == 0 ? 0 : dense_off[lo];
    }
    __syncthreads();
    const long long base0 = carry;
    for (int b0 = lo; b0 < hi; b0 += kSliceBlock) {
        const int idx = b0 + threadIdx.x;
        const long long v = idx < hi ? __ldcg(bytes + idx) : 0;
        const long long inc = warp_incl_scan(v);
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        if (lane == 31) warp_tot[w] = inc;
        __syncthreads();
        if (w == 0) {
            const long long t = warp_incl_scan(lane < kSliceBlock / 32 ? warp_tot[lane] : 0);
            if (lane < kSliceBlock / 32) warp_tot[lane] = t;
        }
        __syncthreads();
        const long long wbase = w > 0 ? warp_tot[w - 1] : 0;
        if (idx < hi) dense_off[idx] = carry + wbase + inc - v;
        __syncthreads();
        if (threadIdx.x == kSliceBlock - 1) carry += wbase + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        dense_off[hi] = carry;
        volatile int64_t* vi = info;
        vi[2 * s] = base0;
        vi[2 * s + 1] = carry - base0;
        __threadfence_system();
    }
}

}  // namespace

int launch_slice_scan(const int32_t* out_bytes, int64_t* dense_off, int32_t lo, int32_t hi,
                      const unsigned* slice_done, int s, int64_t* info, void* stream) {
    k2_slice_scan<<<1, kSliceBlock, 0, static_cast<cudaStream_t>(stream)>>>(out_bytes, dense_off, lo,
                                                                          hi, slice_done, s, info);
    return static_cast<int>(cudaGetLastError());
}

int launch_slice_compact(const uint32_t* scratch, const int64_t* bound_off, const int64_t* dense_off,
                         const int32_t* out_bytes, uint8_t* dense, int32_t lo, int32_t hi,
                         void* stream) {
    if (hi <= lo) return 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int threads = 128;
    long long blocks = (static_cast<long long>(hi - lo) * 32 + threads - 1) / threads;
    if (blocks > 2ll * sms) blocks = 2ll * sms;
    k3_compact<<<static_cast<int>(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(
        scratch, bound_off + lo, dense_off + lo, out_bytes + lo, dense, hi - lo);
    return static_cast<int>(cudaGetLastError());
}

int launch_window_align(int L, const AlignParams& p, int grid, int warps_per_block, void* stream) {
    (void)warps_per_block;
    switch (L) {
        case 1: return launch_L<1>(p, grid, stream);
        case 2: return launch_L<2>(p, grid, stream);
        case 4: return launch_L<4>(p, grid, stream);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

int launch_tail_align(const AlignParams& p, int grid, void* stream) {
    const size_t smem = static_cast<size_t>(band::WARPS) * k1_warp_words<2, true>() * 4;
    cudaError_t e = cudaFuncSetAttribute(k1_tail, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
    k1_tail<<<grid, 32 * band::WARPS, smem, static_cast<cudaStream_t>(stream)>>>(p);
    return static_cast<int>(cudaGetLastError());
}

int launch_mixed_align(int LF, const AlignParams& p, int grid, void* stream) {
    if (LF == 1) return launch_mixed_L<1>(p, grid, stream);
    if (LF == 2) return launch_mixed_L<2>(p, grid, stream);
    return static_cast<int>(cudaErrorInvalidValue);
}

int launch_queue_init(uint32_t* q_band, uint32_t* q_full, uint32_t* q_coop, uint32_t* q_std,
                      unsigned* remaining, int n, const int32_t* n_dev, void* stream) {
    k1_queue_init<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(q_band, q_full, q_coop, q_std,
                                                                  remaining, n, n_dev);
    return static_cast<int>(cudaGetLastError());
}

int mixed_band_warps() { return band::WARPS; }
int mixed_full_warps() { return band::FWARPS; }
int mixed_warps_per_block() { return kMixedWarps; }

int mixed_max_blocks_per_sm(int LF) {
    int blocks = 0;
    cudaError_t e;
    if (LF == 1) {
        const size_t smem = static_cast<size_t>(mixed_block_words<1>()) * 4;
        cudaFuncSetAttribute(k1_mixed<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k1_mixed<1>, 32 * kMixedWarps, smem);
    } else {
        const size_t smem = static_cast<size_t>(mixed_block_words<2>()) * 4;
        cudaFuncSetAttribute(k1_mixed<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k1_mixed<2>, 32 * kMixedWarps, smem);
    }
    return e == cudaSuccess ? blocks : 0;
}

bool band_eligible(int W, int O, int single) {
    return !single && W >= kBandR && W <= band::WMAX && W % kBandR == 0 && W - O >= 1 &&
           W - O <= band::CMAX;
}

size_t bnd_scratch_bytes(int L, long long total_warps) {
    return static_cast<size_t>(total_warps) * static_cast<size_t>(32 * L + 5) * 32 * L * 4;
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
