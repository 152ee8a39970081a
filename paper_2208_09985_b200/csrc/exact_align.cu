// K7 exact_align: the optimal unit-cost global alignment of whole pairs, with
// the reference oracle's tie-breaking (global_align, proj/src/oracle.cpp:39-89),
// hand-written for sm_100a. It replaces the quadratic CPU oracle of the
// accuracy sweep (run_sweep, proj/src/sweep.cpp:40-107).
// Design: DESIGN.md §3.7.
//
//  * DP: Myers' bit-vector algorithm in 32-row blocks of the pattern
//    (vertical deltas Pv/Mv per block, horizontal deltas Ph/Mh, the block's
//    bottom horizontal delta carried to the block below). One warp per pair;
//    lane b owns block b of a 1024-row stripe and runs one column behind
//    lane b-1 (skewed wavefront), receiving the carry and the text code by
//    one shuffle per step. Stripes of a longer pattern run one after another;
//    the bottom carry of each column crosses to the next stripe through a
//    per-pair byte buffer. Row 0 enters with +1 per column (D[i][0] = i).
//  * Every column's Pv/Mv (after) and Ph/Mh (before the shift) are stored,
//    16 B per 32 cells. The traceback from (n, m) recovers D[i-1][j-1],
//    D[i-1][j] and D[i][j-1] from them and applies the forward DP's choice
//    order (diagonal, then delete if strictly better, then insert if strictly
//    better). A match is always the diagonal move, so runs of matches are
//    taken 16 bases at a time from the packed sequences.
//  * The CIGAR bytes ((op << 6) | (len - 1), as K1) are written backwards
//    from the end of the pair's output region and moved to its start, so K2/K3
//    compact them like K1's.
#include "window_align.cuh"

#include <cuda_runtime.h>

namespace sgk {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t bases16(const uint32_t* seq, int64_t a) {
    const int64_t w = a >> 4;
    return __funnelshift_r(__ldcg(seq + w), __ldcg(seq + w + 1), 2 * static_cast<int>(a & 15));
}

__device__ __forceinline__ uint32_t bits32(const uint32_t* m, int64_t a) {
    const int64_t w = a >> 5;
    return __funnelshift_r(__ldcg(m + w), __ldcg(m + w + 1), static_cast<int>(a & 31));
}

__device__ __forceinline__ uint32_t even_bits(uint32_t x) {
    x &= 0x55555555u;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    return (x | (x >> 8)) & 0x0000FFFFu;
}

// 16 mask bits -> the even bits of a 32-bit word (bit k -> bit 2k).
__device__ __forceinline__ uint32_t spread_even(uint32_t s) {
    s &= 0xFFFFu;
    s = (s | (s << 8)) & 0x00FF00FFu;
    s = (s | (s << 4)) & 0x0F0F0F0Fu;
    s = (s | (s << 2)) & 0x33333333u;
    return (s | (s << 1)) & 0x55555555u;
}

// Code of base a: 0..3, or 4 for a non-ACGT base.
__device__ __forceinline__ int base_code(const ExactParams& P, bool hasn, int64_t a) {
    if (hasn && ((__ldcg(P.nmask + (a >> 5)) >> (a & 31)) & 1u)) return 4;
    return static_cast<int>((__ldcg(P.seq + (a >> 4)) >> (2 * (a & 15))) & 3u);
}

__global__ void __launch_bounds__(kThreads) k7_exact_align(const ExactParams P) {
    const int lane = threadIdx.x & 31;
    const long long pair = (static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    if (pair >= P.n_pairs) return;
    const int n = P.text_len[pair], m = P.pat_len[pair];
    const int64_t tb = P.text_off[pair], pb = P.pat_off[pair];
    const bool hasn = P.has_n ? P.has_n[pair] != 0 : false;
    const int nb = (m + 31) >> 5;
    uint4* const st = P.store + P.store_off[pair];  // [nb][n]
    int8_t* const hb = P.hbuf + P.hbuf_off[pair];   // [n]: carries between stripes

    // ---- DP (Myers 1999 blocks; D[i][j] = dist(t[:i], p[:j]))
    for (int k = 0; 32 * k < nb; ++k) {
        const int b = 32 * k + lane;
        const bool act = b < nb;
        const bool more = 32 * (k + 1) < nb;  // a stripe below takes lane 31's carries
        uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0;  // Peq: bit r = pattern base 32b + r is c
        if (act) {
            const int64_t a = pb + 32ll * b;
            const uint32_t w0 = bases16(P.seq, a), w1 = bases16(P.seq, a + 16);
            const uint32_t lo = even_bits(w0) | (even_bits(w1) << 16);
            const uint32_t hi = even_bits(w0 >> 1) | (even_bits(w1 >> 1) << 16);
            const uint32_t ok = hasn ? ~bits32(P.nmask, a) : ~0u;  // N matches nothing
            e0 = ~lo & ~hi & ok;
            e1 = lo & ~hi & ok;
            e2 = ~lo & hi & ok;
            e3 = lo & hi & ok;
        }
        uint32_t pv = ~0u, mv = 0u;  // column 0: D[0][j] = j
        // lane 0: text words / N bits / stripe carries, prefetched 16 columns ahead
        uint32_t tw_cur = 0, tw_nxt = 0, tn_cur = 0, tn_nxt = 0;
        uint4 hc_cur = make_uint4(0, 0, 0, 0), hc_nxt = make_uint4(0, 0, 0, 0);
        if (lane == 0 && n > 0) {
            tw_nxt = bases16(P.seq, tb);
            tn_nxt = hasn ? bits32(P.nmask, tb) : 0u;
            if (k > 0) hc_nxt = *reinterpret_cast<const uint4*>(hb);
        }
        int out = 0;  // to lane + 1: code << 2 | (hout + 1)
        for (int s = 0; s < n + 31; ++s) {
            const int up = __shfl_up_sync(kFull, out, 1);
            const int i = s - lane + 1;  // this lane's column (1-based)
            const bool valid = i >= 1 && i <= n;
            int code = up >> 2, hin = (up & 3) - 1;
            if (lane == 0 && valid) {  // (lane 0 is the only lane whose column is s + 1)
                const int c = i - 1;
                if ((c & 15) == 0) {
                    tw_cur = tw_nxt;
                    tn_cur = tn_nxt;
                    if (c + 16 < n) {
                        tw_nxt = bases16(P.seq, tb + c + 16);
                        tn_nxt = hasn ? bits32(P.nmask, tb + c + 16) : 0u;
                    }
                    if (k > 0) {
                        hc_cur = hc_nxt;
                        if (c + 16 < n) hc_nxt = *reinterpret_cast<const uint4*>(hb + c + 16);
                    }
                }
                code = ((tn_cur >> (c & 15)) & 1u) ? 4 : static_cast<int>((tw_cur >> (2 * (c & 15))) & 3u);
                if (k == 0) {
                    hin = 1;
                } else {
                    const uint32_t w = (c & 15) < 8 ? ((c & 15) < 4 ? hc_cur.x : hc_cur.y)
                                                    : ((c & 15) < 12 ? hc_cur.z : hc_cur.w);
                    hin = static_cast<int>(static_cast<int8_t>((w >> (8 * (c & 3))) & 0xFFu));
                }
            }
            // one column of Myers' block step (the lane's math runs every step;
            // outside its columns the results are dropped)
            uint32_t eq = code == 0 ? e0 : code == 1 ? e1 : code == 2 ? e2 : code == 3 ? e3 : 0u;
            const uint32_t xv = eq | mv;
            eq |= hin < 0 ? 1u : 0u;
            const uint32_t xh = (((eq & pv) + pv) ^ pv) | eq;
            const uint32_t ph = mv | ~(xh | pv);
            const uint32_t mh = pv & xh;
            const int hout = (ph >> 31) ? 1 : ((mh >> 31) ? -1 : 0);
            const uint32_t phs = (ph << 1) | (hin > 0 ? 1u : 0u);
            const uint32_t mhs = (mh << 1) | (hin < 0 ? 1u : 0u);
            const uint32_t pv2 = mhs | ~(xv | phs), mv2 = phs & xv;
            if (valid) {
                pv = pv2;
                mv = mv2;
                if (act) st[static_cast<int64_t>(b) * n + (i - 1)] = make_uint4(pv, mv, ph, mh);
                if (lane == 31 && more) hb[i - 1] = static_cast<int8_t>(hout);
                out = (code << 2) | (hout + 1);
            }
        }
        __syncwarp();  // lane 31's carries and the stored columns are read across lanes next
    }

    // ---- D[n][m] = n + sum of column n's vertical deltas
    int d;
    if (n == 0 || m == 0) {
        d = n + m;
    } else {
        int sum = 0;
        for (int b = lane; b < nb; b += 32) {
            const uint4 w = st[static_cast<int64_t>(b) * n + (n - 1)];
            const int valid = m - 32 * b;
            const uint32_t mask = valid >= 32 ? ~0u : (1u << valid) - 1u;
            sum += __popc(w.x & mask) - __popc(w.y & mask);
        }
        sum = __reduce_add_sync(kFull, static_cast<unsigned>(sum));
        d = n + sum;
    }

    // ---- traceback from (n, m), CIGAR bytes written backwards
    uint8_t* const reg = P.scratch + P.bound_off[pair];
    const int64_t size = ((static_cast<int64_t>(n) + m + 3) & ~int64_t{3}) + 4;
    int64_t pos = size;
    int cur_op = -1, cur_len = 0;
    auto put_byte = [&](int op, int len) {
        --pos;
        if (lane == 0) reg[pos] = static_cast<uint8_t>((op << 6) | (len - 1));
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
        if (cur_op >= 0) put_byte(cur_op, cur_len);
        while (len > 64) {
            put_byte(op, 64);
            len -= 64;
        }
        cur_op = op;
        cur_len = len;
    };
    int i = n, j = m, dd = d;
    while (i > 0 && j > 0) {
        int run = 0;  // matching bases ending at (i-1, j-1); a match is always the diagonal move
        if (i >= 16 && j >= 16) {
            uint32_t x = bases16(P.seq, tb + i - 16) ^ bases16(P.seq, pb + j - 16);
            x = (x | (x >> 1)) & 0x55555555u;  // bit 2k: base k differs
            if (hasn) x |= spread_even(bits32(P.nmask, tb + i - 16) | bits32(P.nmask, pb + j - 16));
            run = __clz(x) >> 1;  // from base 15 (= i-1) downwards
        } else {
            const int lim = min(i, j);
            while (run < lim) {
                const int ct = base_code(P, hasn, tb + i - 1 - run);
                if (ct == 4 || ct != base_code(P, hasn, pb + j - 1 - run)) break;
                ++run;
            }
        }
        if (run > 0) {
            i -= run;
            j -= run;
            emit(0, run);
            continue;
        }
        // mismatch at (i, j): D[i][j-1], D[i-1][j], D[i-1][j-1] from the stored deltas
        const int b = (j - 1) >> 5, r = (j - 1) & 31;
        const uint4 w = st[static_cast<int64_t>(b) * n + (i - 1)];
        const int vi = static_cast<int>((w.x >> r) & 1u) - static_cast<int>((w.y >> r) & 1u);
        const int hi = static_cast<int>((w.z >> r) & 1u) - static_cast<int>((w.w >> r) & 1u);
        int vim1 = 1;  // column 0: D[0][j] - D[0][j-1] = 1
        if (i >= 2) {
            const uint4 w1 = st[static_cast<int64_t>(b) * n + (i - 2)];
            vim1 = static_cast<int>((w1.x >> r) & 1u) - static_cast<int>((w1.y >> r) & 1u);
        }
        const int c = dd - vi, bb = dd - hi, a = bb - vim1;
        int best = a + 1, op = 1;  // substitution
        if (bb + 1 < best) {       // delete text[i-1]
            best = bb + 1;
            op = 3;
        }
        if (c + 1 < best) op = 2;  // insert pattern[j-1]
        if (op == 1) {
            --i;
            --j;
            dd = a;
        } else if (op == 3) {
            --i;
            dd = bb;
        } else {
            --j;
            dd = c;
        }
        emit(op, 1);
    }
    if (i > 0) emit(3, i);  // move[i][0] = delete
    if (j > 0) emit(2, j);  // move[0][j] = insert
    if (cur_op >= 0) put_byte(cur_op, cur_len);
    __syncwarp();
    const int count = static_cast<int>(size - pos);
    for (int o = 0; o < count; o += 32) {  // move to the region start (dst <= src)
        const bool in = o + lane < count;
        const uint8_t v = in ? reg[pos + o + lane] : 0;
        __syncwarp();
        if (in) reg[o + lane] = v;
        __syncwarp();
    }
    if (lane == 0) {
        P.distance[pair] = d;
        P.out_bytes[pair] = count;
    }
}

}  // namespace

int launch_exact_align(const ExactParams& p, void* stream) {
    if (p.n_pairs <= 0) return 0;
    const long long blocks = (static_cast<long long>(p.n_pairs) * 32 + kThreads - 1) / kThreads;
    k7_exact_align<<<static_cast<unsigned>(blocks), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(p);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace sgk
