// K6 wide_align: GenASM-DC + GenASM-TB + window loop for windows wider than
// 128 bits: W in (128, 1024] and single windows of up to 1024 characters
// (BitVector::kMaxBits, proj/include/scrooge/bitvec.hpp:29). Hand-written for
// sm_100a. Design: DESIGN.md §3.6.
//
//  * One warp aligns one pair; lane l holds limb l of every bit vector
//    (32 lanes x 32 bits = 1024). Logical position q = j + 32L - m_w
//    (right-aligned, L = ceil(m_w / 32)) lives in lane q / 32, machine bit
//    31 - q % 32, so the end-of-pattern boundary bit (dp.hpp:145-154) enters
//    at the LSB of lane L-1, and a DP shift is one shuffle (the carry from
//    lane l+1) plus one funnel shift.
//  * DC runs in chunks of 4 rows as a skewed wavefront (row r one column
//    behind row r-1), like K1: the 4 cells of a step are independent. Each
//    row's shifted value serves twice: as its own match term in the next
//    column and as the insertion term of the row below (dp.cpp:187-211 with
//    S(i,d) = I(i+1,d)), so a cell costs one shuffle. The last row of a chunk
//    is parked per column in L2-resident scratch for the next chunk.
//  * Traceback events are the same as K1's, kept in full
//    width for every column the traceback can reach (all columns of a final
//    window, W - O otherwise): X |= R & ~shl1(R[i+1][d]), Y |= R & ~R[i+1][d].
//  * The traceback runs on all lanes in lock step (uniform loads); lane 0
//    writes the run bytes. Outputs are K1's (distance, windows, status, run
//    bytes, counters), so K2/K3 and the host path are shared.
#include "window_align.cuh"

#include <cuda_runtime.h>

#include <cstdio>

namespace sgk {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarps = 4;            // warps per block (independent)
constexpr int kR = 4;                // rows per chunk
constexpr int kTxtWords = 1024 / 4 + 8;  // text codes of a window, 1 byte per column
constexpr int kWarpSmem = 5 * 32 + kTxtWords;  // pattern masks [5][32] + text codes

// R[n][d] of the init column (dp.cpp:146,179): ones(m).shl(min(d, m)), i.e.
// the last d logical positions cleared (positions left of the pattern are
// don't-care). d < 0: all ones.
__device__ __forceinline__ uint32_t init_word(int d, int L, int lane) {
    if (d < 0) return ~0u;
    const int cut = 32 * (L - lane) - d;  // positions p < cut of this limb stay set
    return cut >= 32 ? ~0u : cut <= 0 ? 0u : ~0u << (32 - cut);
}

// shl1 with boundary bit b entering at the end of the pattern (lane L-1).
__device__ __forceinline__ uint32_t shl1(uint32_t x, bool last, bool b) {
    const uint32_t nb = __shfl_down_sync(kFull, x, 1);
    return __funnelshift_l(last ? (b ? 0x80000000u : 0u) : nb, x, 1);
}

// 16 bases (2-bit codes) from base a on, base a in bits 1:0.
__device__ __forceinline__ uint32_t bases16(const uint32_t* seq, int64_t a) {
    const int64_t w = a >> 4;
    return __funnelshift_r(__ldcg(seq + w), __ldcg(seq + w + 1), 2 * static_cast<int>(a & 15));
}

// 32 bits of a 1-bit-per-base mask from base a on.
__device__ __forceinline__ uint32_t bits32(const uint32_t* m, int64_t a) {
    const int64_t w = a >> 5;
    return __funnelshift_r(__ldcg(m + w), __ldcg(m + w + 1), static_cast<int>(a & 31));
}

// Even bits of x packed into the low 16 bits.
__device__ __forceinline__ uint32_t even_bits(uint32_t x) {
    x &= 0x55555555u;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    return (x | (x >> 8)) & 0x0000FFFFu;
}

// 4 two-bit fields (bits 0..7) -> 4 bytes; 4 bits -> 4 bytes of 0/1.
__device__ __forceinline__ uint32_t spread4(uint32_t a) {
    a &= 0xFFu;
    return (a | (a << 6) | (a << 12) | (a << 18)) & 0x03030303u;
}
__device__ __forceinline__ uint32_t spread4bits(uint32_t b) {
    return (b & 1u) | ((b & 2u) << 7) | ((b & 4u) << 14) | ((b & 8u) << 21);
}

// Chunk state. Index 0 is row d0-1 (the parked row of the previous chunk, or
// all ones for d0 = 0); index k = r + 1 is row d0 + r. v: the row's value at
// its current column; vp: at the column before (to its right); sh: shl1(v)
// with the boundary bit of the next column; insp: the insertion term the row
// used at its previous column (its substitution term now); pm: the pattern
// mask of the row's column (handed down the rows with the wavefront).
//
// Scratch is indexed by the step t = S0 - i at which row 0 enters column i,
// in groups of 4 steps: word (t / 4) * 4L + lane * 4 + t % 4 (lanes < L only),
// so that one lane's 4 columns of a group are one 16-byte load or store.
struct Chunk {
    uint32_t v[kR + 1], vp[kR + 1], sh[kR + 1], insp[kR + 1], pm[kR + 1];
    uint32_t ax[4], ay[4];  // events of the 4 columns in flight (slot = entry step % 4)
    uint4 pk0, pk1, pk2;    // parked row: groups g, g+1, g+2 (prefetched two groups ahead)
    uint4 pst, ex, ey;      // row R-1's values / events of the group being completed
    uint32_t pmn;           // pattern mask of row 0's next column
};

template <int C> __device__ __forceinline__ uint32_t& comp(uint4& v) {
    return C == 0 ? v.x : C == 1 ? v.y : C == 2 ? v.z : v.w;
}

struct ChunkGeo {
    int S0, d0, cap, off, L;
    bool last, ors, act;  // lane L-1; OR the events into the earlier chunks'; lane < L
};

#ifdef SG_WIDE_CHECK  // debugging aid: trap on a step outside the warp's scratch
#define SG_COL(c, lo, hi)                                                                  \
    do {                                                                                   \
        if ((c) < (lo) || (c) >= (hi)) {                                                   \
            printf("K6 index %d outside [%d, %d) at line %d\n", (c), (lo), (hi), __LINE__); \
            asm volatile("trap;");                                                         \
        }                                                                                  \
    } while (0)
#else
#define SG_COL(c, lo, hi) do { } while (0)
#endif

// Step variants. kGeneric: any step (rows outside the window skip, the
// d_opt test at column 0, per-row capture test). kMainOut / kMainCap: steps
// with all 4 rows inside the window, none / all of them in the traceback
// columns (the chunk loop picks them per group of 4 steps).
enum { kGeneric = 0, kMainOut = 1, kMainCap = 2 };

// Completes the group of steps t = 4g..4g+3 of row R-1: the parked row (and
// the events: stored in a window's first chunk, OR-ed in later) as one 16-byte
// access per lane.
__device__ __forceinline__ void flush_group(const Chunk& S, const ChunkGeo& G, int g, bool ev,
                                            uint4* park4, uint4* evx4, uint4* evy4) {
    SG_COL(4 * g, 0, G.S0 + 1);
    if (!G.act) return;
    park4[g * G.L] = S.pst;
    if (!ev) return;
    if (!G.ors) {
        evx4[g * G.L] = S.ex;
        evy4[g * G.L] = S.ey;
    } else {  // fire-and-forget reductions: no load of the earlier chunks' events
        unsigned long long* x = reinterpret_cast<unsigned long long*>(evx4 + g * G.L);
        unsigned long long* y = reinterpret_cast<unsigned long long*>(evy4 + g * G.L);
        atomicOr(x, (static_cast<unsigned long long>(S.ex.y) << 32) | S.ex.x);
        atomicOr(x + 1, (static_cast<unsigned long long>(S.ex.w) << 32) | S.ex.z);
        atomicOr(y, (static_cast<unsigned long long>(S.ey.y) << 32) | S.ey.x);
        atomicOr(y + 1, (static_cast<unsigned long long>(S.ey.w) << 32) | S.ey.z);
    }
}

// Step s of a chunk (U = s mod 4, static): rows R-1..0 in descending order
// (each reads its upper neighbour's state from the previous step), the parked
// row advancing just before row 0.
template <int U, int MODE>
__device__ __forceinline__ void chunk_step(Chunk& S, const ChunkGeo& G, int s,
                                           const uint32_t* pmv, const uint8_t* txt,
                                           uint4* park4, uint4* evx4, uint4* evy4, int& fr) {
    constexpr bool GEN = MODE == kGeneric;
    constexpr int CS = (U + 1) & 3;  // row R-1 at step s finishes t = s - 3: component CS
#pragma unroll
    for (int r = kR - 1; r >= 0; --r) {
        const int i = G.S0 - s + r;
        if (r == 0 && (!GEN || s <= G.S0)) {  // the parked row (d0 - 1) moves to column i
            S.vp[0] = S.v[0];
            if (G.d0 > 0) S.v[0] = comp<U>(S.pk0);
            S.sh[0] = G.d0 > 0 ? shl1(S.v[0], G.last, s + 1 > G.d0 - 1) : ~0u;
        }
        if (GEN && (r > s || i < 0)) continue;  // not yet entered / past column 0 (uniform)
        const int k = r + 1;
        const int d = G.d0 + r;
        const int slot = (U - r) & 3;
        if (r > 0) {
            S.pm[k] = S.pm[k - 1];
        } else {
            S.pm[1] = S.pmn;
            S.pmn = !GEN || i >= 1 ? pmv[txt[i - 1] * 32] : ~0u;
        }
        const uint32_t ins = S.sh[k - 1], diag = S.vp[k - 1], sub = S.insp[k];
        const uint32_t se = S.sh[k], east = S.v[k];
        const uint32_t rn = ins & diag & sub & (se | S.pm[k]);  // dp.cpp:187-211
        const bool capt = GEN ? i < G.cap : MODE == kMainCap;
        if (capt) {
            const uint32_t x = rn & ~se, y = rn & ~east;
            if (r == 0) {
                S.ax[slot] = x;
                S.ay[slot] = y;
            } else {
                S.ax[slot] |= x;
                S.ay[slot] |= y;
            }
        }
        S.insp[k] = ins;
        S.vp[k] = east;
        S.v[k] = rn;
        S.sh[k] = shl1(rn, G.last, s - r + 1 > d);  // [n - i > d]
        if (r == kR - 1) {
            comp<CS>(S.pst) = rn;
            if (MODE != kMainOut) {  // (columns left of the traceback region: never read)
                comp<CS>(S.ex) = S.ax[slot];
                comp<CS>(S.ey) = S.ay[slot];
            }
            if (CS == 3) flush_group(S, G, (s - 3) >> 2, MODE != kMainOut, park4, evx4, evy4);
        }
        if (GEN && i == 0 && fr < 0) {  // bit j = 0 of R[0][d] (dp.cpp:222)
            const uint32_t w0 = __shfl_sync(kFull, rn, 0);
            if (!((w0 >> (31 - G.off)) & 1u)) fr = r;
        }
    }
}

// One chunk: rows d0..d0+3 over columns n_w-1..0. Returns the first row r of
// the chunk with bit j = 0 of R[0][d0+r] clear, or -1.
__device__ __noinline__ int dc_chunk(int n_w, int L, int off, bool last, int d0, int cap,
                                     const uint32_t* pmv, const uint8_t* txt, uint4* park4,
                                     uint4* evx4, uint4* evy4, int lane) {
    Chunk S;
    ChunkGeo G{n_w - 1, d0, cap, off, L, last, d0 > 0, lane < L};
#pragma unroll
    for (int k = 0; k <= kR; ++k) {  // every row starts at the init column n
        const int d = d0 + k - 1;
        S.v[k] = init_word(d, L, lane);
        S.vp[k] = S.v[k];
        S.sh[k] = shl1(S.v[k], last, 0 > d);
        S.pm[k] = ~0u;
    }
#pragma unroll
    for (int k = 1; k <= kR; ++k) S.insp[k] = S.sh[k - 1];
    S.insp[0] = ~0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) S.ax[u] = S.ay[u] = 0u;
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    S.pk0 = S.pst = S.ex = S.ey = z;
    S.pk1 = d0 > 0 && G.act ? park4[0] : z;
    S.pk2 = d0 > 0 && G.act ? park4[L] : z;
    S.pmn = pmv[txt[n_w - 1] * 32];
    int fr = -1;
    const int S0 = n_w - 1, nsteps = n_w + kR - 1;
#define SG_GROUP(MODE)                                                    \
    chunk_step<0, MODE>(S, G, s, pmv, txt, park4, evx4, evy4, fr);        \
    chunk_step<1, MODE>(S, G, s + 1, pmv, txt, park4, evx4, evy4, fr);    \
    chunk_step<2, MODE>(S, G, s + 2, pmv, txt, park4, evx4, evy4, fr);    \
    chunk_step<3, MODE>(S, G, s + 3, pmv, txt, park4, evx4, evy4, fr);
    for (int s = 0; s < nsteps; s += 4) {
        if (d0 > 0) {  // parked-row groups g = s/4 (now), g+1, g+2 (prefetch)
            S.pk0 = S.pk1;
            S.pk1 = S.pk2;
            SG_COL(s + 8, 0, S0 + 16);
            if (G.act) S.pk2 = park4[((s >> 2) + 2) * L];  // (past the last group: padding)
        }
        // all rows inside the window and right of column 0 for the whole group
        // (column 0 has the d_opt test): steps 3..S0-1
        const bool full = s >= 3 && s + 3 <= S0 - 1;
        if (full && S0 - (s + 3) >= cap) {
            SG_GROUP(kMainOut)
        } else if (full && S0 - s + 3 < cap) {
            SG_GROUP(kMainCap)
        } else {
            SG_GROUP(kGeneric)
        }
    }
#undef SG_GROUP
    if ((S0 & 3) != 3) flush_group(S, G, S0 >> 2, true, park4, evx4, evy4);  // partial last group
    return fr;
}

// ---------------------------------------------------------------- rows across lane groups
//
// For L <= 8 limbs a single vector leaves lanes idle, so the rows of a chunk
// are spread over the warp instead: G = 32 / LG groups of LG lanes (G = 4, LG = 8),
// group g holding row d0 + g (limb l = lane % LG). The groups form a systolic
// wavefront: at step s group g works on column i = S0 - s + g, receiving the
// upper row's value, its shifted value and the column's event accumulators
// from group g-1 by shuffles (4 per step), and shifting its own value within
// its segment (1 more). Group 0 reads the parked row (value and shifted value)
// from scratch; group G-1 parks its row and stores the column's events. A step
// costs every lane one cell instead of four.
struct GState {
    uint32_t v, sh, dg, insp, ax, ay, pm, pmn;
    uint4 pv0, pv1, pv2, ps0, ps1, ps2;  // parked row / its shift: groups g, g+1, g+2 (group 0)
    uint4 sv, ss, ex, ey;                // group G-1: the t-group being completed
};

struct GGeo {
    int S0, d0, cap, off, L, g, l;
    bool last, act;  // limb L-1; limb < L
};

template <int LG>
__device__ __forceinline__ uint32_t shl1g(uint32_t x, bool last, bool b) {
    const uint32_t nb = __shfl_down_sync(kFull, x, 1, LG);
    return __funnelshift_l(last ? (b ? 0x80000000u : 0u) : nb, x, 1);
}

template <int G>
__device__ __forceinline__ void gflush(const GState& S, const GGeo& Q, int tg, bool ev,
                                       uint4* pv4, uint4* ps4, uint4* evx4, uint4* evy4) {
    if (Q.g != G - 1 || !Q.act) return;
    SG_COL(4 * tg, 0, Q.S0 + 1);
    pv4[tg * Q.L] = S.sv;
    ps4[tg * Q.L] = S.ss;
    if (!ev) return;
    if (Q.d0 == 0) {
        evx4[tg * Q.L] = S.ex;
        evy4[tg * Q.L] = S.ey;
    } else {
        unsigned long long* x = reinterpret_cast<unsigned long long*>(evx4 + tg * Q.L);
        unsigned long long* y = reinterpret_cast<unsigned long long*>(evy4 + tg * Q.L);
        atomicOr(x, (static_cast<unsigned long long>(S.ex.y) << 32) | S.ex.x);
        atomicOr(x + 1, (static_cast<unsigned long long>(S.ex.w) << 32) | S.ex.z);
        atomicOr(y, (static_cast<unsigned long long>(S.ey.y) << 32) | S.ey.x);
        atomicOr(y + 1, (static_cast<unsigned long long>(S.ey.w) << 32) | S.ey.z);
    }
}

template <int G, int U, int MODE>
__device__ __forceinline__ void gstep(GState& S, const GGeo& Q, int s, const uint32_t* pmv,
                                      const uint8_t* txt, uint4* pv4, uint4* ps4, uint4* evx4,
                                      uint4* evy4, int& fr) {
    constexpr int LG = 32 / G;
    constexpr bool GEN = MODE == kGeneric;
    constexpr int CS = (U - (G - 1)) & 3;  // group G-1 finishes t = s - (G-1): component CS
    const int i = Q.S0 - s + Q.g;
    uint32_t nv = __shfl_up_sync(kFull, S.v, LG);
    uint32_t ns = __shfl_up_sync(kFull, S.sh, LG);
    uint32_t nx = __shfl_up_sync(kFull, S.ax, LG);
    uint32_t ny = __shfl_up_sync(kFull, S.ay, LG);
    if (Q.g == 0) {  // row d0 - 1: the parked row (all ones in a window's first chunk)
        nv = Q.d0 > 0 ? comp<U>(S.pv0) : ~0u;
        ns = Q.d0 > 0 ? comp<U>(S.ps0) : ~0u;
        nx = ny = 0u;
    }
    S.pm = S.pmn;
    S.pmn = i >= 1 && i <= Q.S0 + 1 ? pmv[txt[i - 1] * 32] : ~0u;  // next column's mask
    const bool act = !GEN || (s >= Q.g && i >= 0);
    const int d = Q.d0 + Q.g;
    const uint32_t rn = ns & S.dg & S.insp & (S.sh | S.pm);  // dp.cpp:187-211
    const uint32_t shn = shl1g<LG>(rn, Q.last, s + 1 > Q.d0 + 2 * Q.g);  // [n - i > d]
    if (act) {
        const bool capt = GEN ? i < Q.cap : MODE == kMainCap;
        if (capt) {
            S.ax = nx | (rn & ~S.sh);
            S.ay = ny | (rn & ~S.v);
        }
        S.v = rn;
        S.sh = shn;
        comp<CS>(S.sv) = rn;
        comp<CS>(S.ss) = shn;
        if (MODE != kMainOut) {
            comp<CS>(S.ex) = S.ax;
            comp<CS>(S.ey) = S.ay;
        }
    }
    S.dg = nv;  // next column: this column's upper row is the diagonal, its shift the substitution
    S.insp = ns;
    if (CS == 3 && (!GEN || (s - (G - 1) >= 0 && s - (G - 1) <= Q.S0)))
        gflush<G>(S, Q, (s - (G - 1)) >> 2, MODE != kMainOut, pv4, ps4, evx4, evy4);
    (void)d;
    if (GEN) {  // bit j = 0 of R[0][d] when a row reaches column 0 (dp.cpp:222)
        const unsigned hit = __ballot_sync(kFull, act && i == 0 && Q.l == 0 &&
                                                      !((rn >> (31 - Q.off)) & 1u));
        if (hit && fr < 0) fr = s - Q.S0;
    }
}

// One chunk of G rows d0..d0+G-1 (L <= 32 / G). Returns the first row r with
// bit j = 0 of R[0][d0+r] clear, or -1.
template <int G>
__device__ __noinline__ int dc_chunk_g(int n_w, int L, int off, int d0, int cap,
                                       const uint32_t* pmv, const uint8_t* txt, uint4* pv4,
                                       uint4* ps4, uint4* evx4, uint4* evy4, int lane) {
    constexpr int LG = 32 / G;
    const int g = lane / LG, l = lane % LG;
    GGeo Q{n_w - 1, d0, cap, off, L, g, l, l == L - 1, l < L};
    GState S;
    const int d = d0 + g;
    S.v = init_word(d, L, l);  // every row starts at the init column n
    S.sh = shl1g<LG>(S.v, Q.last, 0 > d);
    {   // row 0's diagonal / substitution terms at its first column: R[n][d0-1]
        const uint32_t up = init_word(d0 - 1, L, l);
        const uint32_t ups = shl1g<LG>(up, Q.last, 0 > d0 - 1);
        S.dg = up;
        S.insp = ups;
    }
    S.ax = S.ay = 0u;
    S.pm = ~0u;
    S.pmn = g == 0 ? pmv[txt[n_w - 1] * 32] : ~0u;
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    S.pv0 = S.ps0 = S.sv = S.ss = S.ex = S.ey = z;
    const bool ld = d0 > 0 && g == 0 && Q.act;
    S.pv1 = ld ? pv4[0] : z;
    S.ps1 = ld ? ps4[0] : z;
    S.pv2 = ld ? pv4[L] : z;
    S.ps2 = ld ? ps4[L] : z;
    int fr = -1;
    const int S0 = n_w - 1, nsteps = n_w + G - 1;
#define SG_GGROUP(MODE)                                                            \
    gstep<G, 0, MODE>(S, Q, s, pmv, txt, pv4, ps4, evx4, evy4, fr);                \
    gstep<G, 1, MODE>(S, Q, s + 1, pmv, txt, pv4, ps4, evx4, evy4, fr);            \
    gstep<G, 2, MODE>(S, Q, s + 2, pmv, txt, pv4, ps4, evx4, evy4, fr);            \
    gstep<G, 3, MODE>(S, Q, s + 3, pmv, txt, pv4, ps4, evx4, evy4, fr);
    for (int s = 0; s < nsteps; s += 4) {
        if (ld) {  // parked-row groups s/4 (now), +1, +2 (prefetch; past the end: padding)
            S.pv0 = S.pv1;
            S.pv1 = S.pv2;
            S.ps0 = S.ps1;
            S.ps1 = S.ps2;
            S.pv2 = pv4[((s >> 2) + 2) * L];
            S.ps2 = ps4[((s >> 2) + 2) * L];
        }
        // every group inside the window, none at column 0, for the whole group of steps
        const bool full = s >= G - 1 && s + 3 <= S0 - 1;
        if (full && S0 - (s + 3) >= cap) {
            SG_GGROUP(kMainOut)
        } else if (full && S0 - s + G - 1 < cap) {
            SG_GGROUP(kMainCap)
        } else {
            SG_GGROUP(kGeneric)
        }
    }
#undef SG_GGROUP
    // the last t-group, if partial (t = S0 is completed at step S0 + G - 1)
    if (((S0) & 3) != 3) gflush<G>(S, Q, S0 >> 2, true, pv4, ps4, evx4, evy4);
    return fr;
}

__global__ void __launch_bounds__(32 * kWarps) k6_wide_align(const AlignParams P) {
    extern __shared__ uint32_t smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    uint32_t* const pmv = smem + wib * kWarpSmem;                      // [5][32]
    uint8_t* const txt = reinterpret_cast<uint8_t*>(pmv + 5 * 32);     // [4 kTxtWords]
    uint32_t* const txt32 = pmv + 5 * 32;
    const long long gwarp = static_cast<long long>(blockIdx.x) * kWarps + wib;
    const int wcap = P.wcap;
    uint32_t* const scr = P.bnd + gwarp * static_cast<long long>(wide_warp_words(wcap));
    const int lmax = (wcap + 31) >> 5, wc4 = (wcap + 3) & ~3;  // widest pattern's limbs
    uint32_t* const park = scr;                                             // [wcap + 16 steps][L]
    uint32_t* const parks = park + static_cast<long long>(wc4 + 16) * lmax;  // its shifts (grouped)
    uint32_t* const evx = parks + static_cast<long long>(wc4 + 16) * lmax;  // [wcap + 8 steps][L]
    uint32_t* const evy = evx + static_cast<long long>(wc4 + 8) * lmax;
    pmv[4 * 32 + lane] = ~0u;  // non-ACGT text matches nothing

    const int W = P.W;
    const int step_limit = W - P.O;
    const int K = P.single ? P.k_single : W;  // edit budget: rows 0..K

    for (;;) {
        unsigned q = 0;
        if (lane == 0) q = atomicAdd(P.next_pair, 1u);
        q = __shfl_sync(kFull, q, 0);
        if (q >= static_cast<unsigned>(P.n_pairs)) break;
        const int pair = P.order ? P.order[q] : static_cast<int>(q);
        const int n_tot = P.text_len[pair], m_tot = P.pat_len[pair];
        const int64_t tbase = P.text_off[pair], pbase = P.pat_off[pair];
        {   // streamed upload: wait until the pair's sequence words have arrived
            const int64_t lw = (max(tbase + n_tot, pbase + m_tot) + 15) >> 4;
            const int64_t cw = lw / P.chunk_words;
            const int c = cw < P.n_chunks - 1 ? static_cast<int>(cw) : P.n_chunks - 1;
            while (*reinterpret_cast<const volatile unsigned*>(P.ready + c) == 0u) __nanosleep(1000);
        }
        const bool hasn = P.has_n ? P.has_n[pair] != 0 : false;
        int toff = 0, poff = 0, dist = 0, nwin = 0, status = 0;
        const int window_cap = 4 * ((n_tot + m_tot) / step_limit + 2);  // aligner.cpp:40
        uint32_t* outw = P.scratch + (P.bound_off[pair] >> 2);
        int out_bytes = 0, cur_op = -1, cur_len = 0, acc_n = 0;
        uint32_t acc = 0;
        unsigned long long c_stored = 0, c_writes = 0, c_reads = 0, c_rows = 0, c_cells = 0,
                           c_bequiv = 0;
        // CIGAR run bytes (op << 6) | (len - 1), as in K1 (cigar.cpp:9-16);
        // every lane keeps the same state, lane 0 stores
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

        while (status == 0) {
            // ---- next logical window (aligner.cpp:44-64; single: aligner.cpp:87-112)
            const int n_rem = n_tot - toff, m_rem = m_tot - poff;
            if (n_rem == 0 || m_rem == 0) {
                if (n_rem + m_rem > 0) {  // aligner.cpp:48-57
                    emit(n_rem == 0 ? 2 : 3, n_rem + m_rem);
                    dist += n_rem + m_rem;
                }
                break;
            }
            const bool fin = P.single || (n_rem <= W && m_rem <= W);
            const int n_w = P.single ? n_rem : min(W, n_rem);
            const int m_w = P.single ? m_rem : min(W, m_rem);
            const int limit = fin ? -1 : step_limit;
            const int L = (m_w + 31) >> 5;
            const int off = 32 * L - m_w;
            const bool last = lane == L - 1;
            const int cap = limit < 0 ? n_w : min(n_w, limit);

            // ---- pattern masks (dp.cpp:8-21): bit = 0 iff pattern base == code
            {
                const int js = lane == 0 ? 0 : 32 * lane - off;  // first base of this limb
                const int sh = lane == 0 ? off : 0;               // lane 0: j = 0 sits at p = off
                uint32_t lo = 0u, hi = 0u, nn = ~0u;              // lanes >= L: all ones
                if (lane < L) {
                    const int64_t a = pbase + poff + js;
                    const uint32_t w0 = bases16(P.seq, a), w1 = bases16(P.seq, a + 16);
                    lo = __brev(even_bits(w0) | (even_bits(w1) << 16)) >> sh;
                    hi = __brev(even_bits(w0 >> 1) | (even_bits(w1 >> 1) << 16)) >> sh;
                    nn = hasn ? __brev(bits32(P.nmask, a)) >> sh : 0u;
                    if (sh) nn |= ~(~0u >> sh);  // positions left of the pattern: don't care
                }
                pmv[0 * 32 + lane] = lo | hi | nn;
                pmv[1 * 32 + lane] = ~lo | hi | nn;
                pmv[2 * 32 + lane] = lo | ~hi | nn;
                pmv[3 * 32 + lane] = ~lo | ~hi | nn;
            }
            // ---- text codes, 1 byte per column (non-ACGT -> 4)
            for (int i0 = 16 * lane; i0 < n_w; i0 += 512) {
                const int64_t a = tbase + toff + i0;
                const uint32_t w = bases16(P.seq, a);
                const uint32_t nb = hasn ? bits32(P.nmask, a) : 0u;
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    uint32_t c = spread4(w >> (8 * g));
                    const uint32_t nm = spread4bits(nb >> (4 * g)) * 0xFFu;
                    c = (c & ~nm) | (0x04040404u & nm);
                    txt32[(i0 >> 2) + g] = c;
                }
            }
            __syncwarp();

            // ---- GenASM-DC (dp.cpp:104-231), chunks of 4 rows until d_opt (ET) or row K
            int found_d = -1;
            // L <= 8: the chunk's 4 rows over 4 lane groups of 8; else 4 rows per lane.
            // (Two groups of 16 for L <= 16 measured 2.5x slower than 4 rows per lane
            // at W = 512: half the rows per chunk, and one cell per lane per step
            // leaves the shuffle chain exposed.)
            const int rows = kR;
            for (int d0 = 0;; d0 += rows) {
                int fr;
                if (L <= 8) {
                    uint4* const pv4 = reinterpret_cast<uint4*>(park) + lane % 8;
                    uint4* const ps4 = reinterpret_cast<uint4*>(parks) + lane % 8;
                    uint4* const ex4 = reinterpret_cast<uint4*>(evx) + lane % 8;
                    uint4* const ey4 = reinterpret_cast<uint4*>(evy) + lane % 8;
                    fr = dc_chunk_g<4>(n_w, L, off, d0, cap, pmv + lane % 8, txt, pv4, ps4, ex4,
                                       ey4, lane);
                } else {
                    fr = dc_chunk(n_w, L, off, last, d0, cap, pmv + lane, txt,
                                  reinterpret_cast<uint4*>(park) + lane,
                                  reinterpret_cast<uint4*>(evx) + lane,
                                  reinterpret_cast<uint4*>(evy) + lane, lane);
                }
                if (found_d < 0 && fr >= 0 && d0 + fr <= K) found_d = d0 + fr;
                if ((P.et && found_d >= 0) || d0 + rows > K) break;
            }
            __syncwarp();  // the events are read across lanes below

            // single window with D(0, 0) > k: not found (batch.cpp:57-62)
            const bool not_found = P.single && found_d < 0;
            if (found_d < 0 && !not_found) status = kStInternal | kDetNoStep;  // aligner.cpp:69-70
            {   // reference counters for this window (dp.cpp:23-37,58-75,225-228)
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
            }
            if (not_found) {
                dist = -1;
                ++nwin;
                break;
            }
            if (status) break;

            // ---- GenASM-TB (traceback.cpp:56-113) over the events: runs of
            // matches at once (Match <=> t_i == p_j, both ACGT), at a mismatch
            // Sub > Del > Ins from the events
            int i = 0, j = 0, d = found_d, steps = 0;
            const int lim = limit >= 0 ? limit : 0x3FFFFFFF;
            unsigned reads = 0;
            for (;;) {
                int rem = lim - steps;
                if (rem == 0 || i == n_w || j == m_w) break;
                const int64_t at = tbase + toff + i, ap = pbase + poff + j;
                uint32_t x = bases16(P.seq, at) ^ bases16(P.seq, ap);
                x = (x | (x >> 1)) & 0x55555555u;  // bit 2k: base k differs
                if (hasn) {
                    uint32_t s = (bits32(P.nmask, at) | bits32(P.nmask, ap)) & 0xFFFFu;
                    s = (s | (s << 8)) & 0x00FF00FFu;
                    s = (s | (s << 4)) & 0x0F0F0F0Fu;
                    s = (s | (s << 2)) & 0x33333333u;
                    s = (s | (s << 1)) & 0x55555555u;
                    x |= s;  // non-ACGT bases never match
                }
                const int run = __clz(__brev(x)) >> 1;  // 16 when all 16 bases match
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
                const int qq = j + off;
                const uint32_t bit = 0x80000000u >> (qq & 31);
                const int t = n_w - 1 - i;  // events are stored by entry step
                const int w = (t >> 2) * 4 * L + (qq >> 5) * 4 + (t & 3);
                const uint32_t ex = evx[w], ey = evy[w];
                const int op = ex & bit ? 1 : (ey & bit ? 3 : 2);
                if (d == 0) {
                    status = kStInternal | kDetNoStep;  // traceback.cpp:105-106
                    break;
                }
                reads += 3u;
                i += op != 2;
                j += op != 3;
                --d;
                ++dist;
                ++steps;
                emit(op, 1);
            }
            {   // one side consumed: a single run of indels (traceback.cpp:76-86)
                const int rem = lim - steps;
                if (status == 0 && rem > 0 && !(i == n_w && j == m_w)) {
                    const int op = i == n_w ? 2 : 3;
                    const int left = i == n_w ? m_w - j : n_w - i;
                    if (d != left) status = kStInternal | (i == n_w ? kDetBudgetI : kDetBudgetD);
                    const int k = min(rem, left);
                    i += op != 2 ? k : 0;
                    j += op != 3 ? k : 0;
                    d -= k;
                    dist += k;
                    steps += k;
                    emit(op, k);
                }
            }
            if (!P.single) c_reads += reads;  // single window: counted before TB (aligner.cpp:98-99)
            if (limit < 0 && d != 0 && status == 0) status = kStInternal | kDetLeftover;
            toff += i;
            poff += j;
            ++nwin;
            if (nwin > window_cap) status = kStInternal | kDetWatchdog;
        }

        // ---- finish the pair
        if (cur_op >= 0) put_byte((static_cast<uint32_t>(cur_op) << 6) | (cur_len - 1));
        if (lane == 0) {
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
            if (P.slice_done) {
                __threadfence();
                atomicAdd(P.slice_done + pair / P.slice_pairs, 1u);
            }
        }
        __syncwarp();
    }
}

}  // namespace

size_t wide_smem_bytes() { return static_cast<size_t>(kWarpSmem) * 4 * kWarps; }
int wide_warps_per_block() { return kWarps; }

int wide_max_blocks_per_sm() {
    int blocks = 0;
    cudaFuncSetAttribute(k6_wide_align, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(wide_smem_bytes()));
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &blocks, k6_wide_align, 32 * kWarps, wide_smem_bytes());
    return e == cudaSuccess ? blocks : 0;
}

int launch_wide_align(const AlignParams& p, int grid, void* stream) {
    const size_t smem = wide_smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k6_wide_align, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
    k6_wide_align<<<grid, 32 * kWarps, smem, static_cast<cudaStream_t>(stream)>>>(p);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace sgk
