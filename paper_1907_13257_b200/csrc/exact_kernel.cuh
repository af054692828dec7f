// exact_kernel.cuh — SURVEY.md §8(f) f1: the makespan-optimal schedule of each
// placement ("determining the execution start time of each
// vertex"; constraints :443–453, :465–476), by branch and
// bound, ONE WARP PER PLACEMENT.  DESIGN.md §12.
//
// Nodes F_p / B_p (2K ≤ 64) with the arcs of reading R1; a schedule appends
// nodes one at a time, each starting at max(data ready, its device's free
// time).  Branching is Giffler–Thompson: among the schedulable nodes take y*
// with the least earliest completion c*, on device d*; branch over the
// schedulable nodes of d* whose earliest start is < c* (y* first).  Every
// active schedule is reachable this way, and an optimal schedule can be
// made active, so the minimum over the leaves is the optimum (DESIGN.md §12
// gives the argument).  Bounds (see expand): partial makespan, longest path
// through each unscheduled node with this placement's delays, and each
// device's one-machine bound (earliest start + remaining work + shortest
// tail).
//
// Lane l owns nodes l and l + 32: it tests schedulability (predmask ⊆ S),
// computes est/ect over its arcs, and the warp reduces (ect, node) with
// shuffles and the conflict set with ballots; lanes 0..M−1 evaluate one
// device's one-machine bound each.  The DFS stack, finish times,
// free times and remaining work live in the warp's shared-memory block; the
// warp-uniform control state (S, depth, partial makespan, best) is held
// redundantly in every lane.  Placements are taken from a global counter,
// so warps whose trees are small take more of them.
#pragma once
#include "search_kernel.cuh"

namespace pp {

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
}

// device of π position p of candidate i (same rules as the search kernels)
template <int M, int GEN>
__device__ __forceinline__ uint32_t x_gen_dev(const XParams &P, const uint8_t *orig, uint64_t i, uint32_t p) {
    const uint64_t ii[1] = {i};
    if (GEN == GEN_EXPLICIT) {
        return P.g_place[(i - P.begin) * P.K + orig[p]];
    } else if (GEN == GEN_GRAY) {
        GrayGen<M, 1> g;
        g.init(ii, P.K);
        return Dev<M>::canon(g.dev(0, p, p % 8, 0));
    } else if (GEN == GEN_RANDOM) {
        RandomGen<M, 1> g;
        g.init(i, P.seed, P.K);
        g.refresh(p / 8);
        g.sub((p / 4) & 1);
        return Dev<M>::canon(g.dev(0, p, p % 4, 0));
    } else {
        PerturbGen<M, 1> g;
        g.init(i, P.seed, P.K, P.tau);
        g.refresh(p / 8);
        g.sub((p / 4) & 1);
        return Dev<M>::canon(g.dev(0, p, p % 4, P.g_base[p]));
    }
}

template <int M, int GEN>
__global__ void __launch_bounds__(256) exact_kernel(const XParams P) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t red_mk[8], red_i[8];
    __shared__ bool is_last;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // stage the exact image (plain 16-B loads: a few KB, once per CTA)
    for (uint32_t o = threadIdx.x * 16; o < P.x_bytes; o += blockDim.x * 16)
        *reinterpret_cast<uint4 *>(smem + o) = *reinterpret_cast<const uint4 *>(P.g_ximage + o);
    __syncthreads();
    const XNode *xn = reinterpret_cast<const XNode *>(smem);
    const XPred *xp = reinterpret_cast<const XPred *>(smem + P.off_pred);
    const uint64_t *rows = reinterpret_cast<const uint64_t *>(smem + P.off_rows);
    const uint8_t *cls = smem + P.off_cls;
    const uint64_t *mem = reinterpret_cast<const uint64_t *>(smem + P.off_mem);
    const uint8_t *orig = smem + P.off_orig;
    XWarp &W = *reinterpret_cast<XWarp *>(smem + P.ws_off + warp * sizeof(XWarp));

    const uint32_t N = P.N;
    const uint64_t ALL = (N == 64) ? ~0ull : ((1ull << N) - 1);
    // the lane's two nodes (constant over placements)
    bool own[2];
    uint64_t odur[2], otail[2], opm[2];
    uint32_t opb[2], onp[2], opos[2];
#pragma unroll
    for (int j = 0; j < 2; j++) {
        const uint32_t n = lane + 32 * j;
        own[j] = n < N;
        const XNode x = own[j] ? xn[n] : XNode{};
        odur[j] = x.dur;
        otail[j] = x.tail0;
        opm[j] = x.predmask;
        opb[j] = x.pred_begin;
        onp[j] = x.npred;
        opos[j] = x.pos;
    }

    uint64_t wbest = kInfeasible, wbest_i = ~0ull;   // this warp's argmin (search mode)
    for (;;) {
        uint64_t i = 0;
        if (lane == 0) i = P.begin + atomicAdd(&P.g_work[0], 1ull);
        i = shfl64(i, 0);
        if (i >= P.end) break;
        // an explicit value ≥ M is replaced by device 0 and the row reported
        // infeasible (pp.h, pp_eval_exact): no table is indexed out of range
        bool bad = false;
        // GRAY / GEN_SYM: the placement's packed fields, built once (not per op)
        uint64_t glo = 0, ghi = 0;
        if constexpr (GEN == GEN_GRAY) GrayGen<M, 1>::one(i, P.K, glo, ghi);
        if constexpr (GEN == GEN_SYM) RgsGen<M, 1>::unrank(i, P.K, P.g_rgs, glo, ghi);
        for (uint32_t p = lane; p < P.K; p += 32) {
            uint32_t d;
            if constexpr (GEN == GEN_GRAY || GEN == GEN_SYM) {
                constexpr int b = Bits<M>::b, PF = b ? 64 / b : 64;
                d = M == 1 ? 0u
                           : (uint32_t)((p < (uint32_t)PF ? glo : ghi) >> (p < (uint32_t)PF ? p * b : (p - PF) * b)) &
                                 ((1u << b) - 1);
            } else {
                d = x_gen_dev<M, GEN>(P, orig, i, p);
            }
            bad |= d >= (uint32_t)M;
            W.dev[p] = (uint8_t)(d < (uint32_t)M ? d : 0u);
        }
        bad = __any_sync(0xffffffffu, bad);
        if (lane < 8) {
            W.freeT[lane] = 0;
            W.rem[lane] = 0;
        }
        __syncwarp();
        // remaining work per device and the memory cap (R7)
        bool infeasible = false;
        if (lane < M) {
            uint64_t r = 0, m = 0;
            for (uint32_t n = 0; n < N; n++)
                if (W.dev[xn[n].pos] == lane) r += xn[n].dur;
            for (uint32_t p = 0; p < P.K; p++)
                if (W.dev[p] == lane) m += mem[p];
            W.rem[lane] = r;
            infeasible = P.cap > 0 && m > P.cap;
        }
        infeasible = __any_sync(0xffffffffu, infeasible) || bad;
        uint32_t odev[2];
#pragma unroll
        for (int j = 0; j < 2; j++) odev[j] = own[j] ? W.dev[opos[j]] : 0u;
        // heads and tails with this placement's delays (one lane; node order
        // F_0..F_{K−1}, B_{K−1}..B_0 is topological)
        if (lane == 0) {
            for (uint32_t t = 0; t < N; t++) {
                const uint32_t n = t < P.K ? t : N - 1 - (t - P.K);
                const XNode &x = xn[n];
                const uint32_t dn = W.dev[x.pos];
                uint64_t h = 0;
                for (uint32_t a = 0; a < x.npred; a++) {
                    const XPred q = xp[x.pred_begin + a];
                    const uint32_t dq = W.dev[xn[q.node].pos];
                    const uint64_t v = W.head[q.node] + xn[q.node].dur + rows[q.row * P.xcls + cls[dq * 8 + dn]];
                    h = v > h ? v : h;
                }
                W.head[n] = h;
                W.tail[n] = x.dur;
            }
            for (uint32_t t = N; t-- > 0;) {
                const uint32_t n = t < P.K ? t : N - 1 - (t - P.K);
                const XNode &x = xn[n];
                const uint32_t dn = W.dev[x.pos];
                const uint64_t tn = W.tail[n];
                for (uint32_t a = 0; a < x.npred; a++) {
                    const XPred q = xp[x.pred_begin + a];
                    const uint32_t dq = W.dev[xn[q.node].pos];
                    const uint64_t v = xn[q.node].dur + rows[q.row * P.xcls + cls[dq * 8 + dn]] + tn;
                    if (v > W.tail[q.node]) W.tail[q.node] = v;
                }
            }
        }
        __syncwarp();
        uint64_t ohead[2], otl[2];
#pragma unroll
        for (int j = 0; j < 2; j++) {
            ohead[j] = own[j] ? W.head[lane + 32 * j] : 0;
            otl[j] = own[j] ? W.tail[lane + 32 * j] : 0;
        }
        __syncwarp();

        uint64_t best = kInfeasible;
        bool exact = true;
        if (!infeasible) {
            unsigned long long inc = P.search ? *(volatile unsigned long long *)&P.g_work[1] : ~0ull;
            uint64_t S = 0, pm = 0, nodes = 0;
            int depth = 0;

            // earliest start of one of this lane's nodes (slot j), all preds done
            auto est_of = [&](int j) -> uint64_t {
                const uint32_t dn = j ? odev[1] : odev[0];
                const uint32_t pb = j ? opb[1] : opb[0], np = j ? onp[1] : onp[0];
                uint64_t r = 0;
                for (uint32_t a = 0; a < np; a++) {
                    const XPred q = xp[pb + a];
                    const uint32_t dq = W.dev[xn[q.node].pos];
                    const uint64_t t = W.fin[q.node] + rows[q.row * P.xcls + cls[dq * 8 + dn]];
                    r = t > r ? t : r;
                }
                const uint64_t f = W.freeT[dn];
                return r > f ? r : f;
            };
            // Giffler–Thompson conflict set and the lower bound at state S.
            // Every unscheduled node n starts no earlier than h(n) = its earliest
            // start if schedulable, else max(head(n), free[dev n]); bounds:
            //   path:   max_n h(n) + tail(n)
            //   device: max_d max(free[d], min_{n on d} h(n)) + rem[d]
            //                 + min_{n on d} (tail(n) − Δ(n))
            auto expand = [&](uint64_t &conf, uint32_t &ys, uint64_t &lb) {
                uint64_t e[2], c[2], l = 0;
                bool sch[2];
#pragma unroll
                for (int j = 0; j < 2; j++) {
                    const uint32_t n = lane + 32 * j;
                    const bool un = own[j] && !((S >> n) & 1);
                    sch[j] = un && (opm[j] & ~S) == 0;
                    const uint64_t fr = W.freeT[odev[j]];
                    e[j] = sch[j] ? est_of(j) : (un ? (ohead[j] > fr ? ohead[j] : fr) : kInfeasible);
                    c[j] = sch[j] ? e[j] + odur[j] : kInfeasible;
                    if (un) {
                        const uint64_t b = e[j] + otl[j];
                        l = b > l ? b : l;
                    }
                    if (own[j]) W.ebuf[n] = e[j];
                }
                __syncwarp();
                // lane d < M: the one-machine bound of device d
                if (lane < M) {
                    uint64_t hmin = kInfeasible, tmin = kInfeasible;
                    for (uint32_t n = 0; n < N; n++) {
                        const uint64_t en = W.ebuf[n];
                        if (en != kInfeasible && W.dev[xn[n].pos] == lane) {
                            hmin = en < hmin ? en : hmin;
                            const uint64_t tt = W.tail[n] - xn[n].dur;
                            tmin = tt < tmin ? tt : tmin;
                        }
                    }
                    if (hmin != kInfeasible) {
                        const uint64_t fr = W.freeT[lane];
                        const uint64_t b = (hmin > fr ? hmin : fr) + W.rem[lane] + tmin;
                        l = b > l ? b : l;
                    }
                }
                uint64_t cm = c[0];
                uint32_t cn = lane;
                if (c[1] < cm) { cm = c[1]; cn = lane + 32; }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const uint64_t om = shfl64(cm, lane ^ o);
                    const uint32_t on = __shfl_xor_sync(0xffffffffu, cn, o);
                    const uint64_t ol = shfl64(l, lane ^ o);
                    if (om < cm || (om == cm && on < cn)) { cm = om; cn = on; }
                    l = ol > l ? ol : l;
                }
                ys = cn;
                const uint32_t ds = W.dev[xn[cn].pos];
                const unsigned b0 = __ballot_sync(0xffffffffu, sch[0] && odev[0] == ds && e[0] < cm);
                const unsigned b1 = __ballot_sync(0xffffffffu, sch[1] && odev[1] == ds && e[1] < cm);
                conf = (uint64_t)b0 | ((uint64_t)b1 << 32) | (1ull << cn);
                lb = pm > l ? pm : l;
            };
            auto apply = [&](uint32_t x) {
                const int j = x >> 5;
                const uint64_t s = shfl64(lane == (x & 31) ? est_of(j) : 0, x & 31);
                const XNode &nx = xn[x];
                const uint32_t dx = W.dev[nx.pos];
                const uint64_t f = s + nx.dur;
                if (lane == 0) {
                    W.oldfree[depth] = W.freeT[dx];
                    W.oldpm[depth] = pm;
                    W.chosen[depth] = (uint8_t)x;
                    W.fin[x] = f;
                    W.freeT[dx] = f;
                    W.rem[dx] -= nx.dur;
                }
                S |= 1ull << x;
                pm = f > pm ? f : pm;
                __syncwarp();
            };
            auto undo = [&]() {
                const uint32_t x = W.chosen[depth];
                const XNode &nx = xn[x];
                const uint32_t dx = W.dev[nx.pos];
                pm = W.oldpm[depth];
                __syncwarp();
                if (lane == 0) {
                    W.freeT[dx] = W.oldfree[depth];
                    W.rem[dx] += nx.dur;
                }
                S &= ~(1ull << x);
                __syncwarp();
            };

            uint64_t conf, lb;
            uint32_t ys;
            expand(conf, ys, lb);
            if (P.search && lb > inc) conf = 0;   // cannot win: skip the tree
            if (lane == 0) {
                W.cand[0] = conf;
                W.ystar[0] = (uint8_t)ys;
            }
            __syncwarp();
            for (;;) {
                const uint64_t c = W.cand[depth];
                if (c == 0) {
                    if (depth == 0) break;
                    depth--;
                    undo();
                    continue;
                }
                const uint32_t y = W.ystar[depth];
                const uint32_t x = ((c >> y) & 1) ? y : (uint32_t)(__ffsll((long long)c) - 1);
                __syncwarp();
                if (lane == 0) W.cand[depth] = c & ~(1ull << x);
                apply(x);
                if (++nodes > P.node_limit) { exact = false; break; }
                if (S == ALL) {
                    best = pm < best ? pm : best;
                    undo();
                    continue;
                }
                if (P.search && (nodes & 255) == 0) inc = *(volatile unsigned long long *)&P.g_work[1];
                expand(conf, ys, lb);
                if (lb >= best || (P.search && lb > inc)) {
                    undo();
                    continue;
                }
                depth++;
                if (lane == 0) {
                    W.cand[depth] = conf;
                    W.ystar[depth] = (uint8_t)ys;
                }
                __syncwarp();
            }
        }
        __syncwarp();
        if (lane == 0) {
            if (P.g_makespan) P.g_makespan[i - P.begin] = best;
            if (P.g_exact) P.g_exact[i - P.begin] = exact ? 1 : 0;
            if (!exact) atomicAdd(&P.g_work[2], 1ull);
            if (P.search && exact && best != kInfeasible) atomicMin(&P.g_work[1], (unsigned long long)best);
        }
        // GEN_SYM ranks a relabelling class: its index is the class's smallest
        // Gray index (search_kernel.cuh gray_min_index), needed only when it
        // can still win
        uint64_t key_i = i;
        if constexpr (GEN == GEN_SYM) key_i = best <= wbest ? gray_min_index<M>(glo, ghi, P.K) : kInfeasible;
        if (best < wbest || (best == wbest && key_i < wbest_i)) {
            wbest = best;
            wbest_i = key_i;
        }
    }

    if (!P.search) return;
    // argmin over the CTA, then over CTAs (last-CTA ticket)
    if (lane == 0) {
        red_mk[warp] = wbest;
        red_i[warp] = wbest_i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t m = red_mk[0], ix = red_i[0];
        for (uint32_t w = 1; w < blockDim.x / 32; w++)
            if (lex_less(red_mk[w], red_i[w], m, ix)) { m = red_mk[w]; ix = red_i[w]; }
        P.g_partials[2 * blockIdx.x] = m;
        P.g_partials[2 * blockIdx.x + 1] = ix;
        __threadfence();
        is_last = atomicAdd(P.g_ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last || threadIdx.x != 0) return;
    __threadfence();
    uint64_t m = kInfeasible, ix = ~0ull;
    for (uint32_t b = 0; b < gridDim.x; b++) {
        const uint64_t bm = *(volatile uint64_t *)&P.g_partials[2 * b];
        const uint64_t bi = *(volatile uint64_t *)&P.g_partials[2 * b + 1];
        if (lex_less(bm, bi, m, ix)) { m = bm; ix = bi; }
    }
    P.g_out[0] = m;
    P.g_out[1] = ix;
    P.g_out[2] = *(volatile unsigned long long *)&P.g_work[2];
    *P.g_ticket = 0;
}

template <int M, int GEN>
int launch_exact(const XParams &p, int grid, int threads, int smem, void *stream) {
    exact_kernel<M, GEN><<<grid, threads, smem, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace pp
