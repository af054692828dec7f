// search_kernel.cuh — the hot path: on-device candidate generation, the
// forward+backward in-order list schedule of each candidate placement, and
// the (makespan, index) argmin, for sm_100a.
//
// Kernel shape: LANE PER PLACEMENT.  A warp evaluates 32
// candidate placements in lockstep over the same DFG records, so every record
// read is a warp-uniform shared-memory broadcast; the only per-lane state is
// the finish-time slots ([slot][lane] in shared memory, conflict-free) and the
// per-device free times (registers for M ≤ 2, [device][lane] shared memory
// otherwise).  The recurrence (PAPER.md:443–453 dependency with Δ_e,
// :465–476 one op at a time per device, :497–503 back-to-back + overlapped
// communication; readings R1, R2):
//
//   forward, p in π order:      r = max_{(u,p)} fin[u] + [d_u≠d_p]·c_f
//   backward, p in reverse π:   r = max_{(p,w)} finb[w] + [d_w≠d_p]·c_b
//                               (a sink also waits for its own forward)
//   s = max(r, free[d_p]);  fin = s + Δ;  free[d_p] = fin
//   makespan = max_d free[d]   (memory cap violated ⇒ UINT64_MAX)
//
// The DFG image is staged global → shared once per CTA with a bulk TMA copy
// (cp.async.bulk + mbarrier).  No tensor cores: this is integer max-plus work.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace pp {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    // SplitMix64 finaliser (generator spec)
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

template <int M>
struct Bits {
    static constexpr int b = (M <= 1) ? 0 : (M <= 2) ? 1 : (M <= 4) ? 2 : 3;
};

// ------------------------------------------------------------- generators
// Each generator yields the device of π position p, called with p = 0..K−1
// (forward) and then p = K−1..0 (backward).

template <int M>
struct GrayGen {                           // O5: reflected M-ary Gray code
    static constexpr int b = Bits<M>::b;
    static constexpr int PF = b ? 64 / b : 64;     // fields per register
    uint64_t lo, hi;
    __device__ __forceinline__ void init(uint64_t i, uint32_t K) {
        lo = hi = 0;
        if (M == 1) return;
        if ((M & (M - 1)) == 0) {
            // digits are bit fields; digit j reflects iff a_{j+1} is odd
            for (uint32_t j = 0; j < K; j++) {
                uint64_t a = (j * b < 64) ? (i >> (j * b)) & (M - 1) : 0;
                uint64_t a1 = ((j + 1) * b < 64) ? (i >> ((j + 1) * b)) & 1 : 0;
                uint64_t dj = a1 ? (uint64_t)(M - 1) - a : a;
                if (j < (uint32_t)PF) lo |= dj << (j * b);
                else hi |= dj << ((j - PF) * b);
            }
        } else {
            // general M: even M reflects on a_{j+1} parity, odd M on Σ_{t>j} a_t
            uint64_t a[64];
            uint64_t x = i;
            for (uint32_t j = 0; j < K; j++) { a[j] = x % M; x /= M; }
            uint64_t suffix = 0;   // Σ_{t>j} a_t
            for (int j = (int)K - 1; j >= 0; j--) {
                uint64_t par = (M % 2 == 0) ? ((uint32_t)j + 1 < K ? a[j + 1] : 0) : suffix;
                uint64_t dj = (par & 1) ? (uint64_t)(M - 1) - a[j] : a[j];
                if (j < PF) lo |= dj << (j * b);
                else hi |= dj << ((j - PF) * b);
                suffix += a[j];
            }
        }
    }
    __device__ __forceinline__ uint32_t dev(uint32_t p) const {
        if (M == 1) return 0;
        uint64_t w = (p < (uint32_t)PF) ? lo : hi;
        uint32_t sh = (p < (uint32_t)PF) ? p * b : (p - PF) * b;
        return (uint32_t)(w >> sh) & ((1u << b) - 1);
    }
};

template <int M>
struct RandomGen {                         // O6 RANDOM
    static constexpr int b = Bits<M>::b;
    static constexpr int P = b ? 64 / b : 64;
    uint64_t key;       // seed + γ·(i·Wd + 1)
    uint64_t w;
    uint32_t cur;
    bool zero;
    __device__ __forceinline__ void init(uint64_t i, uint64_t seed, uint32_t K) {
        const uint64_t Wd = (K + P - 1) / P;
        key = seed + 0x9E3779B97F4A7C15ull * (i * Wd + 1);
        zero = (i == 0);
        cur = 0xFFFFFFFFu;
        w = 0;
    }
    __device__ __forceinline__ uint32_t dev(uint32_t p) {
        if (M == 1) return 0;
        uint32_t t = p / P;
        if (t != cur) {   // warp-uniform
            cur = t;
            w = mix64(key + 0x9E3779B97F4A7C15ull * t);
        }
        uint32_t x = (uint32_t)(w >> (b * (p - t * P))) & ((1u << b) - 1);
        uint32_t d = (x * M) >> b;
        return zero ? 0u : d;
    }
};

template <int M>
struct PerturbGen {                        // O6 PERTURB
    static constexpr int b = Bits<M>::b;
    static constexpr int FB = 8 + b;
    static constexpr int P = 64 / FB;
    uint64_t key;
    uint64_t w;
    uint32_t cur;
    uint32_t tau;       // 0 for candidate 0 (the base itself)
    const uint8_t *base;
    __device__ __forceinline__ void init(uint64_t i, uint64_t seed, uint32_t K, uint32_t tau_,
                                         const uint8_t *base_) {
        const uint64_t Wd = (K + P - 1) / P;
        key = (seed ^ 0xD1B54A32D192ED03ull) + 0x9E3779B97F4A7C15ull * (i * Wd + 1);
        tau = (i == 0) ? 0u : tau_;
        cur = 0xFFFFFFFFu;
        w = 0;
        base = base_;
    }
    __device__ __forceinline__ uint32_t dev(uint32_t p) {
        uint32_t bs = base[p];   // uniform broadcast
        if (M == 1) return 0;
        uint32_t t = p / P;
        if (t != cur) {
            cur = t;
            w = mix64(key + 0x9E3779B97F4A7C15ull * t);
        }
        uint32_t f = (uint32_t)(w >> (FB * (p - t * P))) & ((1u << FB) - 1);
        uint32_t u = f & 0xFF, y = f >> 8;
        uint32_t flip = (bs + 1 + (M > 1 ? y % (uint32_t)(M > 1 ? M - 1 : 1) : 0)) % (uint32_t)M;
        return (u >= tau) ? bs : flip;
    }
};

struct ExplicitGen {                       // rows of a [count][K] uint8 array
    const uint8_t *row;
    const uint32_t *orig;
    __device__ __forceinline__ uint32_t dev(uint32_t p) const { return row[orig[p]]; }
};

// ------------------------------------------------------ per-device state
template <int M, bool SMEM>
struct FreeTimes;

template <int M>
struct FreeTimes<M, false> {               // registers, select chains (M ≤ 2)
    uint64_t f[M];
    __device__ __forceinline__ void init(uint64_t *, uint32_t) {
#pragma unroll
        for (int d = 0; d < M; d++) f[d] = 0;
    }
    __device__ __forceinline__ uint64_t get(uint32_t dev) const {
        uint64_t v = f[0];
#pragma unroll
        for (int d = 1; d < M; d++) v = (dev == (uint32_t)d) ? f[d] : v;
        return v;
    }
    __device__ __forceinline__ void set(uint32_t dev, uint64_t v) {
#pragma unroll
        for (int d = 0; d < M; d++) f[d] = (dev == (uint32_t)d) ? v : f[d];
    }
    __device__ __forceinline__ uint64_t max_all() const {
        uint64_t v = f[0];
#pragma unroll
        for (int d = 1; d < M; d++) v = f[d] > v ? f[d] : v;
        return v;
    }
};

template <int M>
struct FreeTimes<M, true> {                // shared memory [device][lane] (M ≥ 3)
    uint64_t *f;
    uint32_t stride;
    __device__ __forceinline__ void init(uint64_t *base, uint32_t s) {
        f = base;
        stride = s;
#pragma unroll
        for (int d = 0; d < M; d++) f[d * stride] = 0;
    }
    __device__ __forceinline__ uint64_t get(uint32_t dev) const { return f[dev * stride]; }
    __device__ __forceinline__ void set(uint32_t dev, uint64_t v) { f[dev * stride] = v; }
    __device__ __forceinline__ uint64_t max_all() const {
        uint64_t v = f[0];
#pragma unroll
        for (int d = 1; d < M; d++) v = f[d * stride] > v ? f[d * stride] : v;
        return v;
    }
};

template <int M>
struct MemUse {
    uint64_t u[M];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int d = 0; d < M; d++) u[d] = 0;
    }
    __device__ __forceinline__ void add(uint32_t dev, uint64_t m) {
#pragma unroll
        for (int d = 0; d < M; d++) u[d] += (dev == (uint32_t)d) ? m : 0;
    }
    // Σ over a device may exceed 2^64 only if Σ M(k) does; saturate
    __device__ __forceinline__ bool over(uint64_t cap) const {
        bool o = false;
#pragma unroll
        for (int d = 0; d < M; d++) o |= u[d] > cap;
        return o;
    }
};

// --------------------------------------------------------- one placement
// Evaluates the schedule of the placement produced by `gen` for this lane.
template <int M, bool MEM, class Gen>
__device__ __forceinline__ uint64_t schedule_one(Gen &gen, const OpRec *__restrict__ ops,
                                                 const EdgeRec *__restrict__ er,
                                                 const uint64_t *__restrict__ mem, uint64_t *slots,
                                                 uint32_t stride, uint64_t *free_base, uint32_t K,
                                                 uint64_t cap) {
    constexpr bool FREE_SMEM = (M > 2);
    FreeTimes<M, FREE_SMEM> fr;
    fr.init(free_base, stride);
    MemUse<M> mu;
    if (MEM) mu.init();

    auto step = [&](uint32_t s, uint32_t p) {
        const OpRec op = ops[s];
        const uint32_t dev = gen.dev(p);
        uint64_t r = 0;
        const uint32_t ne = op.nedge_slot & 0xFFFFu;
        const EdgeRec *e = er + op.edge_begin;
        for (uint32_t q = 0; q < ne; q++) {
            const EdgeRec rec = e[q];
            const uint64_t v = slots[rec.src_slot * stride];
            const uint64_t t = v + ((((uint32_t)v & 7u) != dev) ? rec.c8 : 0ull);
            r = t > r ? t : r;
        }
        const uint64_t f = fr.get(dev);
        const uint64_t st = r > f ? r : f;
        const uint64_t fin = ((st & ~7ull) | dev) + op.cost8;
        slots[(op.nedge_slot >> 16) * stride] = fin;
        fr.set(dev, fin);
        return dev;
    };
    for (uint32_t p = 0; p < K; p++) {
        uint32_t dev = step(p, p);
        if (MEM) mu.add(dev, mem[p]);
    }
    for (uint32_t p = K; p-- > 0;) step(2 * K - 1 - p, p);
    uint64_t mk = fr.max_all() >> 3;
    if (MEM && mu.over(cap)) mk = kInfeasible;
    return mk;
}

__device__ __forceinline__ bool lex_less(uint64_t m1, uint64_t i1, uint64_t m2, uint64_t i2) {
    return m1 < m2 || (m1 == m2 && i1 < i2);
}

// ------------------------------------------------------------------ kernel
template <int M, int GEN, bool MEM, bool WRITE_ALL>
__global__ void __launch_bounds__(256) search_kernel(const KParams P) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint64_t red_mk[8], red_i[8];
    __shared__ bool is_last;

    const uint32_t tid = threadIdx.x;
    const uint32_t lane = tid & 31, warp = tid >> 5;
    const uint32_t nthreads = blockDim.x;

    // ---- stage the image (and the PERTURB base) with bulk TMA copies
    const uint32_t mbar_addr = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_addr));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t total = P.image_bytes + ((GEN == GEN_PERTURB) ? P.base_bytes : 0);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar_addr), "r"(total)
                     : "memory");
        const uint32_t chunk = 32768;
        for (uint32_t off = 0; off < P.image_bytes; off += chunk) {
            uint32_t n = min(chunk, P.image_bytes - off);
            uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem + off);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                "l"(P.g_image + off), "r"(n), "r"(mbar_addr)
                : "memory");
        }
        if (GEN == GEN_PERTURB) {
            uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem + P.smem_base_off);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                "l"(P.g_base), "r"(P.base_bytes), "r"(mbar_addr)
                : "memory");
        }
    }
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                : "=r"(done)
                : "r"(mbar_addr)
                : "memory");
        }
    }

    const OpRec *ops = reinterpret_cast<const OpRec *>(smem);
    const EdgeRec *er = reinterpret_cast<const EdgeRec *>(smem + P.off_edges);
    const uint64_t *mem = reinterpret_cast<const uint64_t *>(smem + P.off_mem);
    const uint32_t *orig = reinterpret_cast<const uint32_t *>(smem + P.off_orig);
    uint64_t *slots = reinterpret_cast<uint64_t *>(smem + P.smem_slots_off) + tid;
    uint64_t *free_base = reinterpret_cast<uint64_t *>(smem + P.smem_free_off) + tid;
    const uint8_t *base = smem + P.smem_base_off;

    uint64_t best_mk = kInfeasible, best_i = kInfeasible;
    bool have = false;
    const uint64_t n = P.end - P.begin;
    const uint64_t ntiles = (n + 31) >> 5;
    const uint64_t wpb = nthreads >> 5;
    for (uint64_t tile = blockIdx.x * wpb + warp; tile < ntiles; tile += (uint64_t)gridDim.x * wpb) {
        const uint64_t off = (tile << 5) + lane;
        const bool valid = off < n;
        const uint64_t i = P.begin + (valid ? off : n - 1);
        uint64_t mk;
        if (GEN == GEN_GRAY) {
            GrayGen<M> g;
            g.init(i, P.K);
            mk = schedule_one<M, MEM>(g, ops, er, mem, slots, nthreads, free_base, P.K, P.cap);
        } else if (GEN == GEN_RANDOM) {
            RandomGen<M> g;
            g.init(i, P.seed, P.K);
            mk = schedule_one<M, MEM>(g, ops, er, mem, slots, nthreads, free_base, P.K, P.cap);
        } else if (GEN == GEN_PERTURB) {
            PerturbGen<M> g;
            g.init(i, P.seed, P.K, P.tau, base);
            mk = schedule_one<M, MEM>(g, ops, er, mem, slots, nthreads, free_base, P.K, P.cap);
        } else {
            ExplicitGen g;
            g.row = P.g_place + (i - P.begin) * (uint64_t)P.K;
            g.orig = orig;
            mk = schedule_one<M, MEM>(g, ops, er, mem, slots, nthreads, free_base, P.K, P.cap);
        }
        if (WRITE_ALL) {
            if (valid) P.g_makespan[off] = mk;
        } else if (valid && (!have || lex_less(mk, i, best_mk, best_i))) {
            best_mk = mk;
            best_i = i;
            have = true;
        }
    }
    if (WRITE_ALL) return;

    // ---- argmin: warp shuffle → CTA (shared) → grid (last CTA)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t om = __shfl_xor_sync(0xffffffffu, best_mk, o);
        uint64_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
        if (lex_less(om, oi, best_mk, best_i)) { best_mk = om; best_i = oi; }
    }
    if (lane == 0) { red_mk[warp] = best_mk; red_i[warp] = best_i; }
    __syncthreads();
    if (tid == 0) {
        for (uint32_t w = 1; w < wpb; w++)
            if (lex_less(red_mk[w], red_i[w], best_mk, best_i)) { best_mk = red_mk[w]; best_i = red_i[w]; }
        P.g_partials[2 * blockIdx.x] = best_mk;
        P.g_partials[2 * blockIdx.x + 1] = best_i;
        __threadfence();
        unsigned t = atomicAdd(P.g_ticket, 1u);
        is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    best_mk = kInfeasible;
    best_i = kInfeasible;
    for (uint32_t c = tid; c < gridDim.x; c += nthreads) {
        uint64_t m = __ldcg(P.g_partials + 2 * c), ii = __ldcg(P.g_partials + 2 * c + 1);
        if (lex_less(m, ii, best_mk, best_i)) { best_mk = m; best_i = ii; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t om = __shfl_xor_sync(0xffffffffu, best_mk, o);
        uint64_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
        if (lex_less(om, oi, best_mk, best_i)) { best_mk = om; best_i = oi; }
    }
    if (lane == 0) { red_mk[warp] = best_mk; red_i[warp] = best_i; }
    __syncthreads();
    if (tid == 0) {
        for (uint32_t w = 1; w < wpb; w++)
            if (lex_less(red_mk[w], red_i[w], best_mk, best_i)) { best_mk = red_mk[w]; best_i = red_i[w]; }
        P.g_out[0] = best_mk;
        P.g_out[1] = best_i;
        *P.g_ticket = 0;   // ready for the next launch on this stream
    }
}

// ---------------------------------------------------------- round update
// One CTA.  Reads the round winner (makespan, index) — the local argmin on one
// GPU, or the NCCL-reduced key/index on several — regenerates its placement,
// keeps the overall best (first round reaching the minimum) and moves the
// PERTURB base to the winner (candidate 0 is the base, so the winner differs
// from the base only when it is strictly better).
template <int M, int GEN>
__global__ void __launch_bounds__(256) round_update_kernel(const UParams U) {
    __shared__ uint64_t mk_s, idx_s;
    __shared__ int improve;
    uint64_t *s = U.s;
    if (threadIdx.x == 0) {
        uint64_t mk, idx;
        if (U.multi) {
            uint64_t key = s[SC_KEY_GLOBAL];
            uint64_t m = key >> 3;
            mk = (m == ((1ull << 61) - 1)) ? kInfeasible : m;
            idx = s[SC_IDX_GLOBAL];
        } else {
            mk = s[SC_LOCAL_MK];
            idx = s[SC_LOCAL_IDX];
        }
        mk_s = mk;
        idx_s = idx;
        improve = (U.round == 0) || (mk < s[SC_BEST_MK]);
    }
    __syncthreads();
    const uint64_t idx = idx_s;
    for (uint32_t p = threadIdx.x; p < U.K; p += blockDim.x) {
        uint32_t d;
        if (GEN == GEN_GRAY) {
            GrayGen<M> g;
            g.init(idx, U.K);
            d = g.dev(p);
        } else if (GEN == GEN_RANDOM) {
            RandomGen<M> g;
            g.init(idx, U.seed, U.K);
            d = g.dev(p);
        } else {
            PerturbGen<M> g;
            g.init(idx, U.seed, U.K, U.tau, U.base);
            d = g.dev(p);
        }
        U.winner[p] = (uint8_t)d;
    }
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < U.K; p += blockDim.x) {
        uint8_t d = U.winner[p];
        if (GEN == GEN_PERTURB) U.base[p] = d;
        if (improve) U.best_place[p] = d;
    }
    if (threadIdx.x == 0 && improve) {
        s[SC_BEST_MK] = mk_s;
        s[SC_BEST_IDX] = idx_s;
        s[SC_BEST_ROUND] = U.round;
    }
}

template <int M, int GEN>
int launch_update(const UParams &u, void *stream) {
    round_update_kernel<M, GEN><<<1, 256, 0, (cudaStream_t)stream>>>(u);
    return (int)cudaGetLastError();
}

template <int M, int GEN, bool MEM, bool WRITE_ALL>
int launch_search(const KParams &p, int grid, int threads, int smem, void *stream) {
    search_kernel<M, GEN, MEM, WRITE_ALL><<<grid, threads, smem, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace pp
