// pipeline.cu — SURVEY.md §8(f) f3: pipeline-parallel MP (GPipe) evaluated
// exhaustively over stage cuts and micro-batch counts (§2;
// PAPER.md:297, §4.4; reading R26 in DESIGN.md §14).
//
// Candidate index = rank·nm + j: rank = the lexicographic rank of the cut
// vector (M−1 increasing π positions in 1..K−1), j = the micro-batch count
// micro[j].  One thread takes a block of consecutive ranks: it unranks the
// first one with a binomial table (shared memory) and steps to the next
// combination after that, so unranking is amortised.  Stage sums come from
// π-prefix sums; the bytes from stage a to stage b from 2-D prefix sums over
// (producer position, consumer position), both L2-resident.  The GPipe row
// recurrences run in registers (M is a template parameter).  The argmin is
// (makespan, index) lexicographic: warp shuffles, CTA, last-CTA ticket.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace pp {

typedef unsigned __int128 u128;

__device__ __forceinline__ uint64_t q2(const uint64_t *Q, uint32_t K1, uint32_t i0, uint32_t i1, uint32_t j0,
                                       uint32_t j1) {
    // Σ over producer positions [i0, i1) and consumer positions [j0, j1)
    return Q[(uint64_t)i1 * K1 + j1] - Q[(uint64_t)i0 * K1 + j1] - Q[(uint64_t)i1 * K1 + j0] +
           Q[(uint64_t)i0 * K1 + j0];
}

__device__ __forceinline__ bool plex_less(uint64_t m1, uint64_t i1, uint64_t m2, uint64_t i2) {
    return m1 < m2 || (m1 == m2 && i1 < i2);
}

// Per-candidate stage-pair values (a < b): forward/backward bytes and their
// per-micro-batch transfer costs.  M ≤ 4 keeps them in registers; M ≥ 5
// (up to 28 pairs × 4 u64) in a per-thread shared-memory column
// [value][pair][thread] after the binomial table, with 128-thread CTAs — in
// registers they needed 255 registers and ~1 KB of spills at M = 8.
template <int M>
constexpr bool kPairsInSmem = M >= 5;
template <int M>
constexpr int kPairs = M * (M - 1) / 2;
template <int M>
__host__ __device__ constexpr int pair_index(int a, int b) {   // a < b
    return a * (2 * M - a - 1) / 2 + (b - a - 1);
}
template <int M>
__host__ __device__ constexpr int pipeline_threads() { return kPairsInSmem<M> ? 128 : 256; }

template <int M, bool SMEM = kPairsInSmem<M>>
struct PairStore {
    uint64_t v[4][kPairs<M> > 0 ? kPairs<M> : 1];
    __device__ __forceinline__ void init(uint64_t *) {}
    __device__ __forceinline__ uint64_t &operator()(int arr, int a, int b) { return v[arr][pair_index<M>(a, b)]; }
};
template <int M>
struct PairStore<M, true> {
    uint64_t *base;
    __device__ __forceinline__ void init(uint64_t *col) { base = col; }
    __device__ __forceinline__ uint64_t &operator()(int arr, int a, int b) {
        return base[(uint32_t)(arr * kPairs<M> + pair_index<M>(a, b)) * pipeline_threads<M>()];
    }
};
enum : int { kDf = 0, kDb = 1, kCf = 2, kCb = 3 };

template <int M>
__global__ void __launch_bounds__(pipeline_threads<M>()) pipeline_kernel(const PipeParams P) {
    extern __shared__ __align__(16) uint64_t binom[];   // [(K+1)·8]: C(n, k), k < 8; then the pair columns
    __shared__ uint64_t red_mk[8], red_i[8];
    __shared__ bool is_last;
    const uint32_t K = P.K, K1 = P.K + 1;
    PairStore<M> pv;
    pv.init(binom + (size_t)K1 * 8 + threadIdx.x);
    for (uint32_t t = threadIdx.x; t < K1 * 8; t += blockDim.x) binom[t] = P.g_binom[t];
    __syncthreads();

    uint64_t bmk = kInfeasible, bidx = ~0ull;
    const uint32_t nm = P.nm;
    const uint64_t r_lo = P.begin / nm, r_hi = (P.end + nm - 1) / nm;   // ranks touching [begin, end)
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (uint64_t r0 = r_lo + tid * P.block; r0 < r_hi; r0 += nthreads * P.block) {
        const uint64_t r1 = min(r_hi, r0 + P.block);
        // unrank r0: cuts[0..M−2] from {1..K−1}, lexicographic
        int32_t cuts[M > 1 ? M - 1 : 1];
        {
            uint64_t rank = r0;
            uint32_t x = 1;
            for (int i = 0; i < M - 1; i++) {
                for (;;) {
                    const uint64_t c = binom[(uint64_t)(K - 1 - x) * 8 + (M - 2 - i)];
                    if (rank < c) break;
                    rank -= c;
                    x++;
                }
                cuts[i] = (int32_t)x;
                x++;
            }
        }
        for (uint64_t r = r0; r < r1; r++) {
            uint32_t st[M + 1];
            st[0] = 0;
            st[M] = K;
#pragma unroll
            for (int s = 1; s < M; s++) st[s] = (uint32_t)cuts[s - 1];
            uint64_t sf[M], sb[M];
            bool infeasible = false;
#pragma unroll
            for (int s = 0; s < M; s++) {
                sf[s] = P.g_pf[st[s + 1]] - P.g_pf[st[s]];
                sb[s] = P.g_pb[st[s + 1]] - P.g_pb[st[s]];
                if (P.cap && P.g_pm[st[s + 1]] - P.g_pm[st[s]] > P.cap) infeasible = true;
            }
            // bytes and edge counts between stages (a < b); has: bit a·8 + b
            uint64_t has = 0;
#pragma unroll
            for (int a = 0; a < M; a++)
#pragma unroll
                for (int b = a + 1; b < M; b++) {
                    const bool h = q2(P.g_qc, K1, st[a], st[a + 1], st[b], st[b + 1]) != 0;
                    has |= (uint64_t)h << (a * 8 + b);
                    pv(kDf, a, b) = h ? q2(P.g_qf, K1, st[a], st[a + 1], st[b], st[b + 1]) : 0;
                    pv(kDb, a, b) = h ? q2(P.g_qb, K1, st[a], st[a + 1], st[b], st[b + 1]) : 0;
                }
            auto has_ab = [&](int a, int b) { return (has >> (a * 8 + b)) & 1; };
            for (uint32_t j = 0; j < nm; j++) {
                const uint64_t idx = r * nm + j;
                if (idx < P.begin || idx >= P.end) continue;
                uint64_t mk = kInfeasible;
                if (!infeasible) {
                    const uint64_t m = P.micro[j];
                    uint64_t tf[M], tb[M];
#pragma unroll
                    for (int s = 0; s < M; s++) {
                        const uint64_t ov = (uint64_t)(st[s + 1] - st[s]) * P.overhead;
                        tf[s] = (sf[s] + m - 1) / m + ov;
                        tb[s] = (sb[s] + m - 1) / m + ov;
                    }
                    const u128 den = (u128)m * P.bw;
#pragma unroll
                    for (int a = 0; a < M; a++)
#pragma unroll
                        for (int b = a + 1; b < M; b++) {
                            if (has_ab(a, b)) {
                                pv(kCf, a, b) = (uint64_t)(((u128)pv(kDf, a, b) * 1000000000000ull + den - 1) / den) + P.lat;
                                pv(kCb, a, b) = (uint64_t)(((u128)pv(kDb, a, b) * 1000000000000ull + den - 1) / den) + P.lat;
                            }
                        }
                    uint64_t F[M], B[M];
#pragma unroll
                    for (int s = 0; s < M; s++) F[s] = 0;
                    for (uint64_t jj = 0; jj < m; jj++) {          // forward, micro-batches in order
#pragma unroll
                        for (int s = 0; s < M; s++) {
                            uint64_t v = F[s];                     // previous micro-batch on device s
#pragma unroll
                            for (int a = 0; a < s; a++)
                                if (has_ab(a, s)) v = max(v, F[a] + pv(kCf, a, s));
                            F[s] = v + tf[s];
                        }
                    }
#pragma unroll
                    for (int s = 0; s < M; s++) B[s] = F[s];       // B[s][m] := F[s][m−1]
                    for (uint64_t jj = 0; jj < m; jj++) {          // backward, micro-batches reversed
#pragma unroll
                        for (int s = M - 1; s >= 0; s--) {
                            uint64_t v = B[s];
#pragma unroll
                            for (int b = s + 1; b < M; b++)
                                if (has_ab(s, b)) v = max(v, B[b] + pv(kCb, s, b));
                            B[s] = v + tb[s];
                        }
                    }
                    mk = 0;
#pragma unroll
                    for (int s = 0; s < M; s++) mk = max(mk, B[s]);
                }
                if (P.g_makespan) P.g_makespan[idx - P.begin] = mk;
                if (plex_less(mk, idx, bmk, bidx)) {
                    bmk = mk;
                    bidx = idx;
                }
            }
            // next combination
            if (M > 1) {
                int i = M - 2;
                while (i >= 0 && cuts[i] == (int32_t)(K - 1 - (M - 2 - i))) i--;
                if (i < 0) break;
                cuts[i]++;
                for (int t = i + 1; t < M - 1; t++) cuts[t] = cuts[t - 1] + 1;
            }
        }
    }
    if (!P.g_out) return;
    // argmin: warp, CTA, grid (last CTA)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t om = __shfl_xor_sync(0xffffffffu, bmk, o);
        const uint64_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (plex_less(om, oi, bmk, bidx)) { bmk = om; bidx = oi; }
    }
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { red_mk[warp] = bmk; red_i[warp] = bidx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t m = red_mk[0], ix = red_i[0];
        for (uint32_t w = 1; w < blockDim.x / 32; w++)
            if (plex_less(red_mk[w], red_i[w], m, ix)) { m = red_mk[w]; ix = red_i[w]; }
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
        if (plex_less(bm, bi, m, ix)) { m = bm; ix = bi; }
    }
    P.g_out[0] = m;
    P.g_out[1] = ix;
    *P.g_ticket = 0;
}

template <int M>
static int launch_m(const PipeParams &p, int grid, int threads, size_t smem, void *stream) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(pipeline_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return (int)e;
    }
    pipeline_kernel<M><<<grid, threads, smem, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

int pipeline_block_threads(int M) {
    switch (M) {
        case 5: return pipeline_threads<5>();
        case 6: return pipeline_threads<6>();
        case 7: return pipeline_threads<7>();
        case 8: return pipeline_threads<8>();
        default: return pipeline_threads<1>();
    }
}

template <int M>
static int launch_m(const PipeParams &p, int grid, void *stream) {
    const size_t smem = (size_t)(p.K + 1) * 8 * sizeof(uint64_t) +
                        (kPairsInSmem<M> ? (size_t)4 * kPairs<M> * pipeline_threads<M>() * sizeof(uint64_t) : 0);
    return launch_m<M>(p, grid, pipeline_threads<M>(), smem, stream);
}

int launch_pipeline(int M, const PipeParams &p, int grid, void *stream) {
    switch (M) {
        case 1: return launch_m<1>(p, grid, stream);
        case 2: return launch_m<2>(p, grid, stream);
        case 3: return launch_m<3>(p, grid, stream);
        case 4: return launch_m<4>(p, grid, stream);
        case 5: return launch_m<5>(p, grid, stream);
        case 6: return launch_m<6>(p, grid, stream);
        case 7: return launch_m<7>(p, grid, stream);
        default: return launch_m<8>(p, grid, stream);
    }
}

}  // namespace pp
