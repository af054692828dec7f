// search_kernel.cuh — the hot path: on-device candidate generation, the
// forward+backward in-order list schedule of each candidate placement, and
// the (makespan, index) argmin, for sm_100a.
//
// Kernel shape: LANE PER PLACEMENT, NP placements per
// lane.  A warp evaluates 32·NP candidate placements in lockstep over the
// same DFG records, so every record read is a warp-uniform shared-memory
// broadcast shared by 32·NP placements.  The recurrence (PAPER.md:443–453
// dependency with Δ_e, :465–476 one op at a time per device, :497–503
// back-to-back ops + overlapped communication; readings R1, R2):
//
//   forward, p in π order:      r = max_{(u,p)} fin[u] + [d_u≠d_p]·c_f
//   backward, p in reverse π:   r = max_{(p,w)} finb[w] + [d_w≠d_p]·c_b
//                               (a sink also waits for its own forward)
//   s = max(r, free[d_p]);  fin = s + Δ;  free[d_p] = fin
//   makespan = max_d free[d]   (memory cap violated ⇒ UINT64_MAX)
//
// Per-placement state: `prev` = the finish time of the previous step (its tag
// is that op's device, so free[tag(prev)] = prev), plus for M = 2 `oth` = the
// free time of the other device (registers), for M ≥ 3 free[] in the warp's
// shared region.  Chain edges (the first input produced by the previous step)
// are read from `prev`; other inputs from liveness-allocated shared slots.
// The schedule loop runs over 8-op groups (one generator word per group),
// each as two half-groups of 4 unrolled steps; K is padded to a multiple of 8
// with state-preserving no-op records.  Three schedule bodies: schedule_gen
// (tagged u64, any M), schedule_f64 (tagged f64, M ≥ 2) and schedule_m2p
// (tagged f64, M = 2 PERTURB — the bench path), which decides the devices and
// cut flags of a half-group at once with SIMD-within-a-register byte compares
// (DESIGN.md §6).
//
// The DFG image is staged global → shared once per CTA with bulk TMA copies
// (cp.async.bulk + mbarrier).  No tensor cores: integer max-plus work.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstddef>
#include <type_traits>

#include "internal.h"

#ifndef PP_CTA_THREADS
#define PP_CTA_THREADS 640   // largest CTA the register allocation targets (A/B: profiles/r01_ab_matrix.txt)
#endif
#ifndef PP_MIN_CTAS
#define PP_MIN_CTAS 1   // resident CTAs per SM the register allocation targets (measured best)
#endif

// max + cost of untagged times on the FP64 pipe (dmax_add) instead of DSETP +
// 2 FSEL + DADD, per code path (A/B: profiles/r01_ab_matrix.txt)
#ifndef PP_FMAX_M2P_CHAIN
#define PP_FMAX_M2P_CHAIN 1   // cut-word schedule, chain steps
#endif
#ifndef PP_FMAX_M2P_JOIN
#define PP_FMAX_M2P_JOIN 0    // cut-word schedule, non-chain steps
#endif
#ifndef PP_FMAX_F64
#define PP_FMAX_F64 2         // schedule_f64: 0 never, 1 always, 2 only PERTURB with M ≥ 3
#endif

namespace pp {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

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
// refresh(g) prepares the 8-op group g (ops 8g..8g+7); dev(k, p, c, base)
// yields the device of π position p = 8g + c for placement k (c is a
// compile-time constant in the unrolled schedule loop).

template <int M, int NP>
struct GrayGen {                           // O5: reflected M-ary Gray code
    static constexpr int b = Bits<M>::b;
    static constexpr int PF = b ? 64 / b : 64;     // fields per register
    uint64_t lo[NP], hi[NP];
    __device__ __forceinline__ static void one(uint64_t i, uint32_t K, uint64_t &lo, uint64_t &hi) {
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
    template <int N>
    __device__ __forceinline__ void init(const uint64_t (&i)[N], uint32_t K) {
#pragma unroll
        for (int k = 0; k < N; k++) one(i[k], K, lo[k], hi[k]);
    }
    __device__ __forceinline__ void refresh(uint32_t) {}
    __device__ __forceinline__ void sub(uint32_t) {}
    __device__ __forceinline__ uint32_t dev(int k, uint32_t p, uint32_t, uint32_t) const {
        if (M == 1) return 0;
        const bool first = p < (uint32_t)PF;
        const uint32_t sh = first ? p * b : (p - PF) * b;
        return (sh < 64) ? (uint32_t)((first ? lo[k] : hi[k]) >> sh) & ((1u << b) - 1) : 0u;
    }
};

// ------------------------- symmetry-reduced exhaustive enumeration (f1)
// With the uniform link model every device is interchangeable: relabelling
// the devices of a placement (a permutation σ of 0..M−1) changes neither its
// schedule's makespan nor its memory feasibility.  An exhaustive GRAY search
// therefore evaluates one placement per class — the restricted-growth string
// (RGS): d[0] = 0 and d[j] ≤ 1 + max(d[0..j−1]), < M — and reports, for the
// classes that reach the running minimum, the smallest Gray index among the
// class's relabellings (gray_min_index), which is the oracle's tie-break over
// all M^K placements.
//
// RGS rank r (lexicographic, d[K−1] fastest) is unranked with the completion
// counts T[rem·kRgsStride + m] = the number of ways to fill `rem` further
// positions when m devices are in use (host-built, pp_dfg::d_rgs): at each
// position the values v < m each cover T[rem][m] ranks, v = m (a new device)
// the next T[rem][m + 1].  The packed fields are GrayGen's, so the schedule
// bodies read them unchanged.
template <int M, int NP>
struct RgsGen : GrayGen<M, NP> {
    using GrayGen<M, NP>::lo;
    using GrayGen<M, NP>::hi;
    static constexpr int b = Bits<M>::b;
    static constexpr int PF = b ? 64 / b : 64;
    // RGS of K positions with rank r into packed fields; returns the number
    // of devices it uses
    __device__ __forceinline__ static uint32_t unrank(uint64_t r, uint32_t K, const uint64_t *__restrict__ T,
                                                      uint64_t &lo, uint64_t &hi) {
        lo = hi = 0;
        if (M == 1) return 1;
        uint32_t m = 1;                                   // d[0] = 0
        for (uint32_t j = 1; j < K; j++) {
            const uint64_t c = __ldg(T + (K - 1 - j) * kRgsStride + m);
            uint32_t v = 0;
            while (v < m && r >= c) { r -= c; v++; }
            if (v == m) m++;                               // opens device m (r < T[rem][m + 1])
            if (j < (uint32_t)PF) lo |= (uint64_t)v << (j * b);
            else hi |= (uint64_t)v << ((j - PF) * b);
        }
        return m;
    }
    __device__ __forceinline__ void init(const uint64_t (&r)[NP], uint32_t K, const uint64_t *T) {
#pragma unroll
        for (int k = 0; k < NP; k++) unrank(r[k], K, T, lo[k], hi[k]);
    }
};

// The smallest Gray index (O5) over the relabellings of placement d (packed
// fields).  Index = Σ a_j·M^j is lexicographic in (a_{K−1}, …, a_0), and
// a_j = d'[j] when the reflection parity of the digits above is even, else
// M − 1 − d'[j].  Going from j = K − 1 down, a device already mapped fixes
// a_j; an unmapped one takes the free target that minimises a_j (the smallest
// free target when even, the largest when odd) — each digit's minimum is
// forced, so the greedy choice is the lexicographic minimum.
template <int M>
__device__ __forceinline__ uint64_t gray_min_index(uint64_t lo, uint64_t hi, uint32_t K) {
    constexpr int b = Bits<M>::b;
    constexpr int PF = b ? 64 / b : 64;
    uint32_t sig = 0xFFFFFFFFu;                           // 4 bits per device label: its target (0xF: unmapped)
    uint32_t used = 0;                                    // targets taken
    uint64_t idx = 0;
    uint32_t par = 0;                                     // a_{j+1} (even M) or Σ_{t>j} a_t (odd M)
    for (int j = (int)K - 1; j >= 0; j--) {
        const uint32_t sh = j < PF ? j * b : (j - PF) * b;
        const uint32_t lab = (uint32_t)((j < PF ? lo : hi) >> sh) & ((1u << b) - 1);
        uint32_t t = (sig >> (4 * lab)) & 0xFu;
        const bool even = (par & 1u) == 0;
        if (t == 0xFu) {
            const uint32_t fr = ~used & ((1u << M) - 1);
            t = even ? (uint32_t)(__ffs((int)fr) - 1) : (uint32_t)(31 - __clz((int)fr));
            used |= 1u << t;
            sig = (sig & ~(0xFu << (4 * lab))) | (t << (4 * lab));
        }
        const uint32_t a = even ? t : (uint32_t)(M - 1) - t;
        idx = idx * (uint64_t)M + a;
        par = (M % 2 == 0) ? a : par + a;
    }
    return idx;
}

// RANDOM and PERTURB keep one key per lane: the lane's placements are
// i_k = i_0 + 32k (search_kernel), so key(i_k) = key(i_0) + k·Δ with the
// uniform Δ = γ·32·Wd, and only i_0 can be candidate 0.  (Per-placement keys
// cost registers that ptxas would rematerialise every group.)
template <int M, int NP>
struct RandomGen {                         // O6 RANDOM: b bits per op, P = 8·⌊8/b⌋ ops per word
    static constexpr int b = Bits<M>::b;
    static constexpr int GPW = b ? 8 / b : 8;      // 8-op groups per word
    uint64_t key0;      // seed + γ·(i_0·Wd + 1)
    uint64_t dk;        // γ·32·Wd
    uint64_t keep0;     // 0 if i_0 is candidate 0 (all zeros), else ~0
    uint64_t w[NP];     // current word
    uint32_t wg[NP];    // the current group's 8·b bits
    uint32_t wh[NP];    // the current half-group's 4·b bits
    uint32_t cur;        // word index held in w (shared by the lane's placements)
    __device__ __forceinline__ void init(uint64_t i0, uint64_t seed, uint32_t K) {
        const uint64_t P = 8ull * GPW;
        const uint64_t Wd = (K + P - 1) / P;
        key0 = seed + kGamma * (i0 * Wd + 1);
        dk = kGamma * 32ull * Wd;
        keep0 = (i0 == 0) ? 0ull : ~0ull;
#pragma unroll
        for (int k = 0; k < NP; k++) {
            w[k] = 0;
            wg[k] = 0;
            wh[k] = 0;
        }
        cur = 0xFFFFFFFFu;
    }
    __device__ __forceinline__ void refresh(uint32_t g) {
        if (M == 1) return;
        const uint32_t t = g / GPW;
        if (t != cur) {   // warp-uniform
            cur = t;
#pragma unroll
            for (int k = 0; k < NP; k++) {
                const uint64_t wk = mix64(key0 + ((uint64_t)k * dk + kGamma * t));
                w[k] = k == 0 ? wk & keep0 : wk;
            }
        }
        const uint32_t sh = 8 * b * (g - t * GPW);
#pragma unroll
        for (int k = 0; k < NP; k++) wg[k] = (uint32_t)(w[k] >> sh);
    }
    // half-group h (ops 8g + 4h .. 8g + 4h + 3)
    __device__ __forceinline__ void sub(uint32_t h) {
#pragma unroll
        for (int k = 0; k < NP; k++) wh[k] = wg[k] >> (4 * b * h);
    }
    // cc = position within the half-group (compile-time in the schedule loop)
    __device__ __forceinline__ uint32_t dev(int k, uint32_t, uint32_t cc, uint32_t) const {
        if (M == 1) return 0;
        const uint32_t x = (wh[k] >> (b * cc)) & ((1u << b) - 1);
        return ((M & (M - 1)) == 0) ? x : (x * M) >> b;
    }
};

template <int M, int NP>
struct PerturbGen {                        // O6 PERTURB (spec revision 3): one byte per op, 8 ops per word
    uint64_t key1, key2;   // the two streams' keys of i_0
    uint64_t dk;           // γ·32·Wd
    uint64_t w[NP], y[NP];
    uint32_t uh[NP], yh[NP];   // the current half-group's u / y bytes
    uint32_t tau0, tau;        // τ of placement 0 (0 if i_0 is candidate 0, the base) and of the others
    __device__ __forceinline__ void init(uint64_t i0, uint64_t seed, uint32_t K, uint32_t tau_) {
        const uint64_t Wd = (K + 7) / 8;
        key1 = (seed ^ 0xD1B54A32D192ED03ull) + kGamma * (i0 * Wd + 1);
        key2 = (seed ^ 0x8CB92BA72F3D8DD7ull) + kGamma * (i0 * Wd + 1);
        dk = kGamma * 32ull * Wd;
        tau = tau_;
        tau0 = (i0 == 0) ? 0u : tau_;
#pragma unroll
        for (int k = 0; k < NP; k++) {
            w[k] = y[k] = 0;
            uh[k] = yh[k] = 0;
        }
    }
    __device__ __forceinline__ void refresh(uint32_t g) {
        if (M == 1) return;
#pragma unroll
        for (int k = 0; k < NP; k++) {
            const uint64_t off = (uint64_t)k * dk + kGamma * g;   // uniform
            w[k] = mix64(key1 + off);
            if (M > 2) y[k] = mix64(key2 + off);
        }
    }
    __device__ __forceinline__ void sub(uint32_t h) {
#pragma unroll
        for (int k = 0; k < NP; k++) {
            uh[k] = h ? (uint32_t)(w[k] >> 32) : (uint32_t)w[k];
            if (M > 2) yh[k] = h ? (uint32_t)(y[k] >> 32) : (uint32_t)y[k];
        }
    }
    // cc = position within the half-group (compile-time in the schedule loop)
    __device__ __forceinline__ uint32_t dev(int k, uint32_t, uint32_t cc, uint32_t bs) const {
        if (M == 1) return 0;
        bs &= 7u;   // bits 7..31 of OpRec.base hold the M = 2 half-group word
        const uint32_t u = __byte_perm(uh[k], 0, 0x4440u | (cc & 3u));
        const uint32_t tk = k == 0 ? tau0 : tau;
        if (M == 2) {
            // device = base + [u < τ], read modulo 2 (see Dev<M>): one PRMT and a sign bit
            return bs + ((uint32_t)((int)u - (int)tk) >> 31);
        }
        const uint32_t yv = __byte_perm(yh[k], 0, 0x4440u | (cc & 3u));
        // revision 3: M = 4, 8 re-draw by XOR; other M move by 1 + y mod (M − 1)
        const uint32_t flip = (M == 4 || M == 8) ? bs ^ (yv & (uint32_t)(M - 1))
                                                 : (bs + 1 + yv % (uint32_t)(M > 1 ? M - 1 : 1)) % (uint32_t)M;
        return (u < tk) ? flip : bs;
    }
};

// A value ≥ M in a row would index free[] out of range (M ≥ 3): it is
// replaced by device 0 and the row is flagged, and a flagged row's makespan
// is PP_INFEASIBLE_MAKESPAN (pp.h, pp_eval_placements).
template <int M, int NP>
struct ExplicitGen {                       // rows of a [count][K] uint8 array
    const uint8_t *row[NP];
    const uint32_t *orig;
    uint32_t bad[NP];
    __device__ __forceinline__ void refresh(uint32_t) {}
    __device__ __forceinline__ void sub(uint32_t) {}
    __device__ __forceinline__ uint32_t dev(int k, uint32_t p, uint32_t, uint32_t) {
        const uint32_t v = row[k][orig[p]];
        const bool ok = v < (uint32_t)M;
        bad[k] |= ok ? 0u : 1u;
        return ok ? v : 0u;
    }
};

// -------------------------------------------------- shared-memory access
// 32-bit shared-window addressing (kept in program order: volatile)
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts64(uint32_t a, uint64_t v) {
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// Memory spaces of the generic schedule body (schedule_gen): the shared-
// memory tier addresses the image and the lane state by 32-bit shared-window
// addresses; the global-state tier (DFGs whose image or per-lane state does
// not fit in shared memory, search_big_kernel) by 64-bit global addresses,
// with the same [slot][lane] layout (a warp's 32 lanes read 256 contiguous
// bytes) — records through the read-only path, state through L1/L2.
struct SmemSpace {
    typedef uint32_t Addr;
    static __device__ __forceinline__ uint4 rec(Addr a) { return lds128(a); }
    static __device__ __forceinline__ uint64_t ld(Addr a) { return lds64(a); }
    static __device__ __forceinline__ void st(Addr a, uint64_t v) { sts64(a, v); }
    static __device__ __forceinline__ double ldd(Addr a) { return __longlong_as_double((long long)lds64(a)); }
    static __device__ __forceinline__ void std(Addr a, double v) { sts64(a, (uint64_t)__double_as_longlong(v)); }
    static __device__ __forceinline__ uint32_t ld32(Addr a) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
        return v;
    }
};
struct GmemSpace {
    typedef uint64_t Addr;
    static __device__ __forceinline__ uint4 rec(Addr a) { return __ldg(reinterpret_cast<const uint4 *>(a)); }
    static __device__ __forceinline__ uint64_t ld(Addr a) { return *reinterpret_cast<const uint64_t *>(a); }
    static __device__ __forceinline__ void st(Addr a, uint64_t v) { *reinterpret_cast<uint64_t *>(a) = v; }
    static __device__ __forceinline__ double ldd(Addr a) { return *reinterpret_cast<const double *>(a); }
    static __device__ __forceinline__ void std(Addr a, double v) { *reinterpret_cast<double *>(a) = v; }
    static __device__ __forceinline__ uint32_t ld32(Addr a) { return __ldg(reinterpret_cast<const uint32_t *>(a)); }
};
// An extra input's record by one LDS.128 (default) or by two loads, its cost
// as an aligned double (LDS.64) and its slot offset (LDS.32), which saves the
// two register moves into an aligned pair (PP_EXTRA_SPLIT=1).  A/B
// (profiles/r02_ab_extra.txt): M = 2 ±0.3%, GNMT M = 4 +0.25%, Inception
// M = 4 −1.0%, so not adopted.
#ifndef PP_EXTRA_SPLIT
#define PP_EXTRA_SPLIT 0
#endif

// ---------------------------------------------------------- arithmetic
// Two exact representations of a tagged finish time (internal.h):
//   ArithU64: 8·t + device in a u64;
//   ArithF64: t + device·ulp(t) in a double, t < 2^49 (adds and compares on
//             the FP64 pipe instead of the INT32 ALU pipe).
struct ArithU64 {
    typedef uint64_t V;
    static __device__ __forceinline__ V from_bits(uint64_t b) { return b; }
    static __device__ __forceinline__ uint64_t to_bits(V v) { return v; }
    static __device__ __forceinline__ uint32_t lo(V v) { return (uint32_t)v; }
    static __device__ __forceinline__ V add(V v, uint64_t c) { return v + c; }
    static __device__ __forceinline__ V vmax(V a, V b) { return a > b ? a : b; }
    static __device__ __forceinline__ V finish(V s, uint32_t dev, uint64_t cost) { return ((s & ~7ull) | dev) + cost; }
    static __device__ __forceinline__ uint64_t ps(V v) { return v >> 3; }
};

struct ArithF64 {
    typedef double V;
    static __device__ __forceinline__ V from_bits(uint64_t b) { return __longlong_as_double((long long)b); }
    static __device__ __forceinline__ uint64_t to_bits(V v) { return (uint64_t)__double_as_longlong(v); }
    static __device__ __forceinline__ uint32_t lo(V v) { return (uint32_t)__double2loint(v); }
    static __device__ __forceinline__ V add(V v, uint64_t c) { return __dadd_rn(v, from_bits(c)); }
    static __device__ __forceinline__ V vmax(V a, V b) { return a > b ? a : b; }
    // ((s with the tag cleared) + cost) with the tag set to dev
    static __device__ __forceinline__ V finish(V s, uint32_t dev, uint64_t cost) {
        const double t = __hiloint2double(__double2hiint(s), __double2loint(s) & ~7);
        const double x = __dadd_rn(t, from_bits(cost));
        return __hiloint2double(__double2hiint(x), __double2loint(x) | (int)dev);
    }
    static __device__ __forceinline__ uint64_t ps(V v) {
        return (uint64_t)__double2ull_rz(__hiloint2double(__double2hiint(v), __double2loint(v) & ~7));
    }
};

// For M = 2 a device is any integer read modulo 2 (the PERTURB generator
// yields base + flip ∈ {0, 1, 2}); tags compare on bit 0 only.  Otherwise
// devices are 0..M−1 and tags compare on the 3 tag bits.
template <int M>
struct Dev {
    static constexpr uint32_t mask = (M == 2) ? 1u : 7u;
    static __device__ __forceinline__ uint32_t canon(uint32_t d) { return d & mask; }
};
template <class A, int M>
__device__ __forceinline__ bool same_dev(typename A::V v, uint32_t dev) {
    return ((A::lo(v) ^ dev) & Dev<M>::mask) == 0;
}
// v + (tag(v) ≠ dev ? c : 0): the cut-edge charge
template <class A, int M>
__device__ __forceinline__ typename A::V cut_add(typename A::V v, uint32_t dev, uint64_t c) {
    return same_dev<A, M>(v, dev) ? v : A::add(v, c);
}

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
    __device__ __forceinline__ bool over(uint64_t cap) const {
        bool o = false;
#pragma unroll
        for (int d = 0; d < M; d++) o |= u[d] > cap;
        return o;
    }
};

// -------------------------------------------------- NP placements per lane
// lane: address of this lane's entry in its warp region (region + 8·lane);
// placement k's copy of a slot is at +k·256.  S: the memory space of the
// image and the state (SmemSpace, or GmemSpace for the global-state tier).
template <int M, int NP, bool MEM, bool F64, class Gen, class S = SmemSpace>
__device__ __forceinline__ void schedule_gen(Gen &gen, uint64_t (&mk)[NP], typename S::Addr ops, typename S::Addr xr,
                                            const uint64_t *__restrict__ mem, typename S::Addr lane, uint32_t free_off,
                                            uint32_t K8, uint64_t cap) {
    typedef typename S::Addr Addr;
    typedef typename std::conditional<F64, ArithF64, ArithU64>::type A;
    typedef typename A::V V;
    V prev[NP], oth[NP];
    MemUse<M> mu[NP];
#pragma unroll
    for (int k = 0; k < NP; k++) {
        prev[k] = A::from_bits(0);
        oth[k] = A::from_bits(0);
        if (MEM) mu[k].init();
        if (M > 2) {
#pragma unroll
            for (int d = 0; d < M; d++) S::st(lane + free_off * NP + d * NP * 256 + k * 256, 0);
        }
    }
    Addr x = xr;

    auto step = [&](Addr rec, uint32_t p, uint32_t c, bool fwd) {
        const uint4 a = S::rec(rec);
        const uint4 b = S::rec(rec + 16);
        const uint64_t cost = ((uint64_t)a.y << 32) | a.x;
        const uint64_t c0 = ((uint64_t)a.w << 32) | a.z;
        uint32_t dev[NP];
#pragma unroll
        for (int k = 0; k < NP; k++) dev[k] = gen.dev(k, p, c, b.w);
        if (M <= 2 && b.z == 0) {
            // fast path: the only input is the previous step's output (a chain edge)
#pragma unroll
            for (int k = 0; k < NP; k++) {
                V s;
                if (M == 1) {
                    s = prev[k];
                } else if (F64) {
                    // x = 1 iff the chain edge is cut (then free[dev] = oth),
                    // x = 0 iff dev = tag(prev) (then free[dev] = prev).  With
                    // cut = (double)x and same = 1 − cut, all exact:
                    //   t = prev + cut·c0,  f = oth − same·2^50 (< 0 if same),
                    //   s = max(t, f),      oth' = cut·prev + same·oth
                    const uint32_t xbit = (A::lo(prev[k]) ^ dev[k]) & 1u;
                    const double cut = __hiloint2double((int)(xbit * 0x3FF00000u), 0);
                    const double same = __hiloint2double((int)((1u - xbit) * 0x3FF00000u), 0);
                    const double pv = reinterpret_cast<const double &>(prev[k]);
                    const double ov = reinterpret_cast<const double &>(oth[k]);
                    const double t = __fma_rn(__longlong_as_double((long long)c0), cut, pv);
                    const double f = __fma_rn(same, -1125899906842624.0, ov);
                    const double sv = t > f ? t : f;
                    const double on = __fma_rn(cut, pv, __dmul_rn(same, ov));
                    s = reinterpret_cast<const V &>(sv);
                    oth[k] = reinterpret_cast<const V &>(on);
                } else {
                    const bool same = same_dev<A, M>(prev[k], dev[k]);   // also: not a cut edge
                    const V m = A::vmax(A::add(prev[k], c0), oth[k]);
                    s = same ? prev[k] : m;
                    oth[k] = same ? oth[k] : prev[k];
                }
                prev[k] = A::finish(s, dev[k], cost);
            }
        } else {
            V r[NP];
            if (b.x == kFromPrev) {
#pragma unroll
                for (int k = 0; k < NP; k++) r[k] = cut_add<A, M>(prev[k], dev[k], c0);
            } else {
#pragma unroll
                for (int k = 0; k < NP; k++) r[k] = cut_add<A, M>(A::from_bits(S::ld(lane + b.x * NP + k * 256)), dev[k], c0);
            }
            const uint32_t nx = b.z & 0xFFFFu;
#pragma unroll 1
            for (uint32_t q = 0; q < nx; q++) {   // further inputs (uniform trip count)
                const uint4 e = S::rec(x);
                x += sizeof(ExtraRec);
                const uint64_t ce = ((uint64_t)e.y << 32) | e.x;
#pragma unroll
                for (int k = 0; k < NP; k++)
                    r[k] = A::vmax(r[k], cut_add<A, M>(A::from_bits(S::ld(lane + e.z * NP + k * 256)), dev[k], ce));
            }
#pragma unroll
            for (int k = 0; k < NP; k++) {
                V s;
                if (M == 1) {
                    s = A::vmax(r[k], prev[k]);
                } else if (M == 2) {
                    const bool same = same_dev<A, M>(prev[k], dev[k]);
                    s = A::vmax(r[k], same ? prev[k] : oth[k]);
                    oth[k] = same ? oth[k] : prev[k];
                } else {
                    const Addr fa = lane + free_off * NP + dev[k] * NP * 256 + k * 256;
                    s = A::vmax(r[k], A::from_bits(S::ld(fa)));
                    prev[k] = A::finish(s, dev[k], cost);
                    S::st(fa, A::to_bits(prev[k]));
                    continue;
                }
                prev[k] = A::finish(s, dev[k], cost);
            }
        }
        if (b.y != kNoStore) {
#pragma unroll
            for (int k = 0; k < NP; k++) S::st(lane + b.y * NP + k * 256, A::to_bits(prev[k]));
        }
        if (MEM && fwd) {
            const uint64_t m = mem[p];
#pragma unroll
            for (int k = 0; k < NP; k++) mu[k].add(Dev<M>::canon(dev[k]), m);
        }
    };
    // the two half-groups of an 8-op group: looped at NP = 4 (the unrolled
    // body overflows the instruction cache), unrolled below (A/B measured)
    constexpr int kHalfUnroll = NP >= 4 ? 1 : 2;
    const uint32_t G = K8 / 8;
    for (uint32_t g = 0; g < G; g++) {           // forward, π order
        gen.refresh(g);
#pragma unroll (kHalfUnroll)
        for (uint32_t h = 0; h < 2; h++) {
            gen.sub(h);
            const Addr rec = ops + (g * 8 + h * 4) * (uint32_t)sizeof(OpRec);
#pragma unroll
            for (uint32_t cc = 0; cc < 4; cc++) step(rec + cc * (uint32_t)sizeof(OpRec), g * 8 + h * 4 + cc, cc, true);
        }
    }
    for (uint32_t g = G; g-- > 0;) {             // backward, reverse π order
        gen.refresh(g);
#pragma unroll (kHalfUnroll)
        for (uint32_t h = 2; h-- > 0;) {
            gen.sub(h);
            const Addr rec = ops + (2 * K8 - 1 - g * 8 - h * 4) * (uint32_t)sizeof(OpRec);
#pragma unroll
            for (int cc = 3; cc >= 0; cc--)
                step(rec - (Addr)cc * (Addr)sizeof(OpRec), g * 8 + h * 4 + cc, cc, false);
        }
    }
#pragma unroll
    for (int k = 0; k < NP; k++) {
        V v;
        if (M <= 2) {
            v = A::vmax(prev[k], oth[k]);
        } else {
            v = A::from_bits(0);
#pragma unroll
            for (int d = 0; d < M; d++) v = A::vmax(v, A::from_bits(S::ld(lane + free_off * NP + d * NP * 256 + k * 256)));
        }
        mk[k] = A::ps(v);
        if (MEM && mu[k].over(cap)) mk[k] = kInfeasible;
    }
}

#ifndef PP_BIG_REC_PREFETCH
#define PP_BIG_REC_PREFETCH 1   // global tier: next record loaded one step ahead (A/B: profiles/r02_big_bench_prefetch.txt)
#endif
// ------------------------------------------------ tagged-f64 specialisation
// State per placement: prev = finish time of the previous step as an exact
// integer double (UNTAGGED), pdev = its device, and the other devices' free
// times: M = 2 — `oth` in a register; M ≥ 3 — free[d] in the warp's shared
// region, where free[pdev] may be stale (≤ prev) because the live value is
// prev.  Slot values stay tagged (t + d·ulp(t)) for the non-chain reads; the
// tag is set only when a value is stored.  With cut = [dev ≠ pdev] ∈ {0.0,
// 1.0}, a chain step is
//   s = max(prev + cut·c0, cut·free[dev])   (no cut: free[dev] is prev, and
//                                            cut·free = 0 ≤ prev drops out)
//   prev' = s + cost, pdev' = dev, and the old prev becomes free[pdev]:
//   M = 2: oth' = oth + cut·(prev − oth);  M ≥ 3: free[pdev] ← prev (always)
// — every operation exact on integers < 2^49; only the max needs a select.
// x ∈ {0,1} → 0.0 / 1.0 as one IMAD on the FMA pipe: khi = 0x3FF00000 (the
// high word of 1.0) is a kernel parameter, so ptxas cannot turn the multiply
// into an ISETP + SEL pair on the ALU pipe.
__device__ __forceinline__ double one_if(uint32_t x, uint32_t khi) {
    uint32_t hi;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(hi) : "r"(x), "r"(khi));
    return __hiloint2double((int)hi, 0);
}
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
// max(a, b) + c for UNTAGGED exact integers a, b, c < 2^49 on the FP64 pipe:
// ½·(a + b + |a − b|) + c — a + b and |a − b| are exact (< 2^50), their sum
// is 2·max(a, b) (< 2^51, even), and the fused ½·x + c is the exact integer
// max + c < 2^50.  Four FP64 instructions instead of DSETP, 2 FSEL (ALU pipe)
// and DADD (A/B: profiles/r01_ab_matrix.txt).
__device__ __forceinline__ double dmax_add(double a, double b, double c) {
    return __fma_rn(0.5, __dadd_rn(__dadd_rn(a, b), fabs(__dadd_rn(a, -b))), c);
}
__device__ __forceinline__ double with_tag(double v, uint32_t dev) {
    return __hiloint2double(__double2hiint(v), __double2loint(v) | (int)dev);
}
__device__ __forceinline__ double clear_tag(double v) {
    return __hiloint2double(__double2hiint(v), __double2loint(v) & ~7);
}
__device__ __forceinline__ double ldd(uint32_t a) { return __longlong_as_double((long long)lds64(a)); }
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void std_(uint32_t a, double v) { sts64(a, (uint64_t)__double_as_longlong(v)); }

template <int M>
__device__ __forceinline__ uint32_t cut_bit(uint32_t a, uint32_t b) {   // 1 iff devices differ
    return (M == 2) ? ((a ^ b) & 1u) : (uint32_t)(((a ^ b) & 7u) != 0);
}
// v + [tag(v) ≠ dev]·c for a tagged slot value
// 1.0 iff devices a and b differ, else 0.0.  M = 2: (a ⊕ b) & 1 times the
// high word of 1.0 (LOP3 + IMAD); M ≥ 3: a select on the 3-bit compare
// (LOP3 with a predicate + SEL; PP_CUT_SEL=0 keeps the 0/1 multiply, A/B)
#ifndef PP_CUT_SEL
#define PP_CUT_SEL 1
#endif
template <int M>
__device__ __forceinline__ double cut_one(uint32_t a, uint32_t b, uint32_t khi) {
    if (M == 2 || !PP_CUT_SEL) return one_if(cut_bit<M>(a, b), khi);
    return __hiloint2double((int)((((a ^ b) & 7u) != 0) ? khi : 0u), 0);
}
template <int M>
__device__ __forceinline__ double cut_add_f64(double v, uint32_t dev, double c, uint32_t khi) {
    return __fma_rn(c, cut_one<M>((uint32_t)__double2loint(v), dev, khi), v);
}

// Hardware graph (HW): a record's cost field is the image offset of its cost
// row; the transfer a → b costs row[cls[a][b]], class 0 (a = b) costing 0, so
// an input is simply v + row[cls[tag(v)][dev]] (no cut flag needed).
template <int M, int NP, bool MEM, bool HW, class Gen, class S = SmemSpace>
__device__ __forceinline__ void schedule_f64(Gen &gen, uint64_t (&mk)[NP], typename S::Addr ops, typename S::Addr xr,
                                             const uint64_t *__restrict__ mem, typename S::Addr lane,
                                             uint32_t free_off, uint32_t K8, uint64_t cap, uint32_t khi, uint32_t cls,
                                             uint32_t hq = 0, uint32_t nslot = 0) {
    typedef typename S::Addr Addr;
    static_assert(!HW || std::is_same<S, SmemSpace>::value, "hardware graphs run on the shared tier");
    constexpr bool SM = M > 2;                    // free[] in shared memory
    // Gray prefix reuse (GEN_SYM): the lane's NP placements are
    // consecutive RGS ranks, identical on the first hq forward half-groups
    // (warp-uniform), which are computed for placement 0 only; its state
    // (registers and the nslot live slots) is then copied to the others
    constexpr bool kPrefix = std::is_same<Gen, RgsGen<M, NP>>::value && NP > 1;
    constexpr bool kFmax = PP_FMAX_F64 == 1 || (PP_FMAX_F64 == 2 && SM && std::is_same<Gen, PerturbGen<M, NP>>::value);
    double prev[NP], oth[NP];
    uint32_t pdev[NP];
    MemUse<M> mu[NP];
#pragma unroll
    for (int k = 0; k < NP; k++) {
        prev[k] = 0.0;
        oth[k] = 0.0;
        pdev[k] = 0;
        if (MEM) mu[k].init();
        if (SM) {
#pragma unroll
            for (int d = 0; d < M; d++) S::std(lane + free_off * NP + d * NP * 256 + k * 256, 0.0);
        }
    }
    auto fslot = [&](int k, uint32_t d) -> Addr { return lane + free_off * NP + d * NP * 256 + k * 256; };
    auto hwc = [&](uint32_t row, uint32_t a, uint32_t b) {   // cost of a transfer a → b
        return S::ldd(ops + row + 8 * lds8(cls + Dev<M>::canon(a) * 8 + Dev<M>::canon(b)));
    };
    Addr x = xr;

    // global tier (GmemSpace): records are consumed strictly in address order
    // (forward π, then the backward records), so the next step's
    // record is loaded when a step starts, off the L1 latency of the next one.
    // With two placements per lane (M ≤ 2) only: at NP = 1 (M ≥ 3) the extra
    // registers spill (A/B: profiles/r02_big_bench_prefetch.txt)
    constexpr bool kRecPrefetch = std::is_same<S, GmemSpace>::value && PP_BIG_REC_PREFETCH && NP >= 2;
    uint4 na = {0, 0, 0, 0}, nb = {0, 0, 0, 0};
    if constexpr (kRecPrefetch) {
        na = S::rec(ops);
        nb = S::rec(ops + 16);
    }
    auto step = [&](auto KNc, Addr rec, uint32_t p, uint32_t c, bool fwd) {
        constexpr int KN = decltype(KNc)::value;   // placements 0..KN−1 (KN < NP: the shared prefix)
        uint4 a, b;
        if constexpr (kRecPrefetch) {
            a = na;
            b = nb;
            na = S::rec(rec + sizeof(OpRec));        // past the last record: the extras (unused)
            nb = S::rec(rec + sizeof(OpRec) + 16);
        } else {
            a = S::rec(rec);
            b = S::rec(rec + 16);
        }
        const double cost = __hiloint2double((int)a.y, (int)a.x);
        const double c0 = __hiloint2double((int)a.w, (int)a.z);
        uint32_t dev[NP];
#pragma unroll
        for (int k = 0; k < KN; k++) dev[k] = gen.dev(k, p, c, b.w);
        if (b.z == 0) {
            // chain step: the only input is the previous step's output
#pragma unroll
            for (int k = 0; k < KN; k++) {
                // free[dev] matters only across a cut (else it is prev, and
                // cut·free = 0 ≤ prev): s = max(prev + cut·c0, cut·free[dev])
                const double cut = cut_one<M>(pdev[k], dev[k], khi);
                const double t = HW ? __dadd_rn(prev[k], hwc(a.z, pdev[k], dev[k])) : __fma_rn(c0, cut, prev[k]);
                double f;
                if (SM) {
                    // free[dev] is exact across a cut; without one it is
                    // free[pdev]'s stale shared copy, ≤ prev ≤ t, so the max
                    // is t either way and no cut factor is needed
                    f = S::ldd(fslot(k, dev[k]));
                    S::std(fslot(k, pdev[k]), prev[k]);
                } else {
                    f = __dmul_rn(cut, oth[k]);
                    oth[k] = __fma_rn(cut, __dadd_rn(prev[k], -oth[k]), oth[k]);   // cut ? prev : oth
                }
                prev[k] = kFmax ? dmax_add(t, f, cost) : __dadd_rn(dmax(t, f), cost);
                pdev[k] = dev[k];
            }
        } else {
            double r[NP];
            if (b.x == kFromPrev) {
#pragma unroll
                for (int k = 0; k < KN; k++)
                    r[k] = HW ? __dadd_rn(prev[k], hwc(a.z, pdev[k], dev[k]))
                              : __fma_rn(c0, cut_one<M>(pdev[k], dev[k], khi), prev[k]);
            } else {
#pragma unroll
                for (int k = 0; k < KN; k++) {
                    const double v = S::ldd(lane + b.x * NP + k * 256);
                    r[k] = HW ? __dadd_rn(v, hwc(a.z, (uint32_t)__double2loint(v) & 7u, dev[k]))
                              : cut_add_f64<M>(v, dev[k], c0, khi);
                }
            }
            const uint32_t nx = b.z & 0xFFFFu;
#pragma unroll 1
            for (uint32_t q = 0; q < nx; q++) {   // further inputs (uniform trip count)
                double ce;
                uint32_t ex, ez;
                if (PP_EXTRA_SPLIT && !HW) {
                    ce = S::ldd(x);
                    ez = S::ld32(x + 8);
                    ex = 0;
                } else {
                    const uint4 e = S::rec(x);
                    ce = __hiloint2double((int)e.y, (int)e.x);
                    ex = e.x;
                    ez = e.z;
                }
                x += sizeof(ExtraRec);
#pragma unroll
                for (int k = 0; k < KN; k++) {
                    const double v = S::ldd(lane + ez * NP + k * 256);
                    r[k] = dmax(r[k], HW ? __dadd_rn(v, hwc(ex, (uint32_t)__double2loint(v) & 7u, dev[k]))
                                         : cut_add_f64<M>(v, dev[k], ce, khi));
                }
            }
#pragma unroll
            for (int k = 0; k < KN; k++) {
                // free[dev] = cut ? other : prev, exact on the FP64 pipe
                const double cut = cut_one<M>(pdev[k], dev[k], khi);
                double f;
                if (SM) {
                    f = __fma_rn(cut, __dadd_rn(S::ldd(fslot(k, dev[k])), -prev[k]), prev[k]);
                    S::std(fslot(k, pdev[k]), prev[k]);
                } else {
                    const double d = __dadd_rn(prev[k], -oth[k]);
                    f = __fma_rn(-cut, d, prev[k]);
                    oth[k] = __fma_rn(cut, d, oth[k]);
                }
                prev[k] = kFmax ? dmax_add(clear_tag(r[k]), f, cost) : __dadd_rn(clear_tag(dmax(r[k], f)), cost);
                pdev[k] = dev[k];
            }
        }
        if (b.y != kNoStore) {
#pragma unroll
            for (int k = 0; k < KN; k++) S::std(lane + b.y * NP + k * 256, with_tag(prev[k], Dev<M>::canon(dev[k])));
        }
        if (MEM && fwd) {
            const uint64_t m = mem[p];
#pragma unroll
            for (int k = 0; k < KN; k++) mu[k].add(Dev<M>::canon(dev[k]), m);
        }
    };
    // the two half-groups of an 8-op group: looped at NP = 4 (the unrolled
    // body overflows the instruction cache), unrolled below (A/B measured)
    constexpr int kHalfUnroll = NP >= 4 ? 1 : 2;
    using All = std::integral_constant<int, NP>;
    const uint32_t G = K8 / 8;
    uint32_t g0 = 0, h0 = 0;
    if constexpr (kPrefix) {
        using One = std::integral_constant<int, 1>;
        for (uint32_t hg = 0; hg < hq; hg++) {   // the shared prefix, placement 0 only
            const uint32_t g = hg >> 1, h = hg & 1;
            if (h == 0) gen.refresh(g);
            gen.sub(h);
            const Addr rec = ops + (g * 8 + h * 4) * (uint32_t)sizeof(OpRec);
#pragma unroll
            for (uint32_t cc = 0; cc < 4; cc++)
                step(One{}, rec + cc * (uint32_t)sizeof(OpRec), g * 8 + h * 4 + cc, cc, true);
        }
        if (hq) {
#pragma unroll
            for (int k = 1; k < NP; k++) {
                prev[k] = prev[0];
                oth[k] = oth[0];
                pdev[k] = pdev[0];
                if (MEM) mu[k] = mu[0];
            }
            for (uint32_t sl = 0; sl < nslot; sl++) {
                const double v = S::ldd(lane + sl * NP * 256);
#pragma unroll
                for (int k = 1; k < NP; k++) S::std(lane + sl * NP * 256 + k * 256, v);
            }
            if (SM) {
#pragma unroll
                for (int d = 0; d < M; d++) {
                    const double v = S::ldd(fslot(0, d));
#pragma unroll
                    for (int k = 1; k < NP; k++) S::std(fslot(k, d), v);
                }
            }
        }
        g0 = hq >> 1;
        h0 = hq & 1;
    }
    for (uint32_t g = g0; g < G; g++) {          // forward, π order
        gen.refresh(g);
#pragma unroll (kHalfUnroll)
        for (uint32_t h = 0; h < 2; h++) {
            if (kPrefix && g == g0 && h < h0) continue;
            gen.sub(h);
            const Addr rec = ops + (g * 8 + h * 4) * (uint32_t)sizeof(OpRec);
#pragma unroll
            for (uint32_t cc = 0; cc < 4; cc++)
                step(All{}, rec + cc * (uint32_t)sizeof(OpRec), g * 8 + h * 4 + cc, cc, true);
        }
    }
    for (uint32_t g = G; g-- > 0;) {             // backward, reverse π order
        gen.refresh(g);
#pragma unroll (kHalfUnroll)
        for (uint32_t h = 2; h-- > 0;) {
            gen.sub(h);
            const Addr rec = ops + (2 * K8 - 1 - g * 8 - h * 4) * (uint32_t)sizeof(OpRec);
#pragma unroll
            for (int cc = 3; cc >= 0; cc--)
                step(All{}, rec - (Addr)cc * (Addr)sizeof(OpRec), g * 8 + h * 4 + cc, cc, false);
        }
    }
#pragma unroll
    for (int k = 0; k < NP; k++) {
        double v = prev[k];
        if (SM) {
#pragma unroll
            for (int d = 0; d < M; d++) v = dmax(v, S::ldd(fslot(k, d)));   // stale free[pdev] ≤ prev
        } else {
            v = dmax(v, oth[k]);
        }
        mk[k] = (uint64_t)__double2ull_rz(v);
        if (MEM && mu[k].over(cap)) mk[k] = kInfeasible;
    }
}

// ------------------------------- M = 2 PERTURB: cut words (tagged f64)
// The same schedule as schedule_f64<2> for the PERTURB generator, with the
// devices of a half-group (4 ops) decided at once.  Per placement and
// half-group, with the 4 PERTURB bytes u_c of the half-group in one word:
//   flip_c = [u_c < τ]                  — 4 byte compares in 4 SIMD-within-a-
//                                          register ops (bit 7 of byte c)
//   dev_c  = flip_c ⊕ base_c            — the packed base word of the image
//   cut_c  = dev_c ⊕ dev of the previous scheduled step   (one PRMT, one XOR)
// and per step the cut flag is widened to a full-word mask by one PRMT
// (sign replication of byte c).  The byte compare, with τ' = τ (τ ≤ 128) or
// τ − 128 (τ > 128) in every byte and x = (u | 0x80…) − τ' (no borrow crosses
// a byte; bit 7 of byte c of x is [u_c mod 128 ≥ τ']):
//   τ ≤ 128:  u_c < τ  ⟺  ¬(u_c,7 ∨ x_c,7)
//   τ > 128:  u_c < τ  ⟺  ¬(u_c,7 ∧ x_c,7)
// — both ¬MAJ(u, x, A) with A = all ones (τ ≤ 128) or zero (τ > 128).
// Candidate 0 (the base) masks its flips to zero.  The arithmetic is
// schedule_f64's, operation for operation; only the cut flags are derived
// differently, so the results are identical (the parity suite checks both).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}

// m = all ones ? a : b, word by word (LOP3 on the ALU pipe)
__device__ __forceinline__ double dsel(uint32_t m, double a, double b) {
    return __hiloint2double((int)lop3<0xCA>(m, (uint32_t)__double2hiint(a), (uint32_t)__double2hiint(b)),
                            (int)lop3<0xCA>(m, (uint32_t)__double2loint(a), (uint32_t)__double2loint(b)));
}
#ifndef PP_M2P_SEL
#define PP_M2P_SEL 1   // oth / free[dev] by mask selects (ALU; A/B: -1.4% time) instead of DADD + DFMA (FP64)
#endif
#ifndef PP_M2P_LDS64
#define PP_M2P_LDS64 1   // cost and c0 by two LDS.64 into their own pairs (A/B: -1.1%)
#endif
#ifndef PP_DYN_TILES
#define PP_DYN_TILES 1   // argmin kernels take tiles from a global counter (0: static stride, for A/B)
#endif
#ifndef PP_MPW_PREFETCH
#define PP_MPW_PREFETCH 1   // schedule_mpw: free[dev] of the next step loaded one step ahead (A/B)
#endif
#ifndef PP_TILE_PREFETCH
#define PP_TILE_PREFETCH 0   // dynamic tiles: claim the next tile when a tile starts (A/B)
#endif
#ifndef PP_M2P_MIX
#define PP_M2P_MIX 0   // chain steps: placements k with k % 4 < MIX take the ALU max (DSETP + 2 FSEL) instead of dmax_add (pipe balance)
#endif
#ifndef PP_M2P_CUTIMAD
#define PP_M2P_CUTIMAD 0   // 1: the cut flag's high word by IMAD (FMA pipe) instead of LOP3 (ALU)
#endif
#ifndef PP_M2P_STEPLOOP
#define PP_M2P_STEPLOOP 0   // 1: the 4 steps of a half-group as a loop (smaller code) instead of unrolled
#endif

// The PERTURB words of this lane's placements i_k =
// i_0 + 32k: word g of placement i is mix64(key(i) + γ·g) with key(i) =
// (seed ⊕ C1) + γ·(i·Wd + 1), i.e. mix64(A_g + k·Δ) with A_g = key(i_0) + γ·g
// (one running 64-bit value per lane) and Δ = γ·32·Wd (uniform).
template <int NP, bool MEM, bool RP = false>
__device__ __forceinline__ void schedule_m2p(uint64_t A, uint64_t dA, uint32_t hk0, uint64_t (&mk)[NP], uint32_t ops,
                                             uint32_t xr, const uint64_t *__restrict__ mem, uint32_t lane, uint32_t K8,
                                             uint64_t cap, uint32_t khi, uint32_t tau) {
    constexpr uint32_t H = 0x80808080u;
    const uint32_t tq = (tau <= 128 ? tau : tau - 128) * 0x01010101u;
    const uint32_t amaj = tau <= 128 ? ~0u : 0u;
    double prev[NP], oth[NP];
    uint32_t dw[NP], cw[NP], dprev[NP];
    uint64_t w[NP];
    MemUse<2> mu[NP];
#pragma unroll
    for (int k = 0; k < NP; k++) {
        prev[k] = 0.0;
        oth[k] = 0.0;
        dprev[k] = 0;                  // device 0 before the first step (schedule_f64's pdev = 0)
        dw[k] = cw[k] = 0;
        w[k] = 0;
        if (MEM) mu[k].init();
    }
    uint32_t x = xr;
    auto refresh = [&]() {
#pragma unroll
        for (int k = 0; k < NP; k++) w[k] = mix64(A + (uint64_t)k * dA);
    };

    // the device and cut words of half-group h of the current group, whose
    // records carry the packed base word `bw`
    auto half = [&](uint32_t h, uint32_t bw, bool fwd) {
        const uint32_t bsw = bw & H;
#pragma unroll
        for (int k = 0; k < NP; k++) {
            const uint32_t u = h ? (uint32_t)(w[k] >> 32) : (uint32_t)w[k];
            const uint32_t y = (u | H) - tq;
            const uint32_t mj = lop3<0xE8>(u, y, amaj);                 // MAJ(u, y, A)
            dw[k] = lop3<0x9A>(k == 0 ? hk0 : H, mj, bsw);            // (hk ∧ ¬mj) ⊕ bsw
            // the previous scheduled step's device, byte-aligned with dev_c:
            // forward (c − 1; c = 0 takes byte 3 of the previous half-group),
            // backward (c + 1; c = 3 takes byte 0 of the previous half-group)
            const uint32_t sh = fwd ? prmt(dw[k], dprev[k], 0x2107u) : prmt(dw[k], dprev[k], 0x4321u);
            cw[k] = dw[k] ^ sh;
            dprev[k] = dw[k];
        }
    };

    // records are read in address order: with RP the next step's record is
    // loaded when a step starts (used when few warps are resident; as
    // schedule_mpw, profiles/r02_ab_rec_prefetch.txt)
    double rcost = 0.0, rc0 = 0.0;
    uint4 rb = {0, 0, 0, 0};
    if constexpr (RP) {
        rcost = ldd(ops);
        rc0 = ldd(ops + 8);
        rb = lds128(ops + 16);
    }
    auto step = [&](uint32_t rec, uint32_t p, uint32_t c, bool fwd) {
        uint4 a, b;
        double cost, c0;
        if constexpr (RP) {
            cost = rcost;
            c0 = rc0;
            b = rb;
            rcost = ldd(rec + sizeof(OpRec));
            rc0 = ldd(rec + sizeof(OpRec) + 8);
            rb = lds128(rec + sizeof(OpRec) + 16);
        } else if (PP_M2P_LDS64) {
            cost = ldd(rec);
            c0 = ldd(rec + 8);
            b = lds128(rec + 16);
        } else {
            a = lds128(rec);
            b = lds128(rec + 16);
            cost = __hiloint2double((int)a.y, (int)a.x);
            c0 = __hiloint2double((int)a.w, (int)a.z);
        }
        uint32_t m[NP];
        double cut[NP];
#pragma unroll
        for (int k = 0; k < NP; k++) {
            m[k] = prmt(cw[k], 0u, 0x8888u | (c * 0x1111u));    // all ones iff cut_c
            cut[k] = PP_M2P_CUTIMAD ? __hiloint2double((int)(m[k] * (0u - khi)), 0)   // −1·−khi = khi
                                    : __hiloint2double((int)(m[k] & khi), 0);        // 1.0 or 0.0
        }
        if (b.z == 0) {
            // chain step: s = max(prev + cut·c0, cut·oth), oth' = cut ? prev : oth
#pragma unroll
            for (int k = 0; k < NP; k++) {
                const double t = __fma_rn(c0, cut[k], prev[k]);
                const double f = __dmul_rn(cut[k], oth[k]);
                if (PP_M2P_SEL) oth[k] = dsel(m[k], prev[k], oth[k]);
                else oth[k] = __fma_rn(cut[k], __dadd_rn(prev[k], -oth[k]), oth[k]);
                const bool alu_max = (k % 4) < PP_M2P_MIX;
                prev[k] = (PP_FMAX_M2P_CHAIN && !alu_max) ? dmax_add(t, f, cost) : __dadd_rn(dmax(t, f), cost);
            }
        } else {
            double r[NP];
            if (b.x == kFromPrev) {
#pragma unroll
                for (int k = 0; k < NP; k++) r[k] = __fma_rn(c0, cut[k], prev[k]);
            } else {
#pragma unroll
                for (int k = 0; k < NP; k++)
                    r[k] = cut_add_f64<2>(ldd(lane + b.x * NP + k * 256), dw[k] >> (8 * c + 7), c0, khi);
            }
            const uint32_t nx = b.z & 0xFFFFu;
#pragma unroll 1
            for (uint32_t q = 0; q < nx; q++) {   // further inputs (uniform trip count)
                double ce;
                uint32_t ez;
                if (PP_EXTRA_SPLIT) {
                    ce = ldd(x);
                    ez = lds32(x + 8);
                } else {
                    const uint4 e = lds128(x);
                    ce = __hiloint2double((int)e.y, (int)e.x);
                    ez = e.z;
                }
                x += sizeof(ExtraRec);
#pragma unroll
                for (int k = 0; k < NP; k++)
                    r[k] = dmax(r[k], cut_add_f64<2>(ldd(lane + ez * NP + k * 256), dw[k] >> (8 * c + 7), ce, khi));
            }
#pragma unroll
            for (int k = 0; k < NP; k++) {
                // free[dev] = cut ? oth : prev
                double f;
                if (PP_M2P_SEL) {
                    f = dsel(m[k], oth[k], prev[k]);
                    oth[k] = dsel(m[k], prev[k], oth[k]);
                } else {
                    const double d = __dadd_rn(prev[k], -oth[k]);
                    f = __fma_rn(-cut[k], d, prev[k]);
                    oth[k] = __fma_rn(cut[k], d, oth[k]);
                }
                prev[k] = PP_FMAX_M2P_JOIN ? dmax_add(clear_tag(r[k]), f, cost) : __dadd_rn(clear_tag(dmax(r[k], f)), cost);
            }
        }
        if (b.y != kNoStore) {
#pragma unroll
            for (int k = 0; k < NP; k++) std_(lane + b.y * NP + k * 256, with_tag(prev[k], (dw[k] >> (8 * c + 7)) & 1u));
        }
        if (MEM && fwd) {
            const uint64_t mm = mem[p];
#pragma unroll
            for (int k = 0; k < NP; k++) mu[k].add((dw[k] >> (8 * c + 7)) & 1u, mm);
        }
    };
    constexpr int kHalfUnroll = NP >= 4 ? 1 : 2;
    constexpr int kStepUnroll = PP_M2P_STEPLOOP ? 1 : 4;
    const uint32_t G = K8 / 8;
    for (uint32_t g = 0; g < G; g++) {           // forward, π order
        refresh();
        A += kGamma;
#pragma unroll (kHalfUnroll)
        for (uint32_t h = 0; h < 2; h++) {
            const uint32_t rec = ops + (g * 8 + h * 4) * (uint32_t)sizeof(OpRec);
            half(h, lds32(rec + offsetof(OpRec, base)), true);
#pragma unroll (kStepUnroll)
            for (uint32_t cc = 0; cc < 4; cc++) step(rec + cc * (uint32_t)sizeof(OpRec), g * 8 + h * 4 + cc, cc, true);
        }
    }
#pragma unroll
    for (int k = 0; k < NP; k++) dprev[k] >>= 24;   // byte 0 := the device of the last forward step
    for (uint32_t g = G; g-- > 0;) {             // backward, reverse π order
        A -= kGamma;
        refresh();
#pragma unroll (kHalfUnroll)
        for (uint32_t h = 2; h-- > 0;) {
            const uint32_t rec = ops + (2 * K8 - 1 - g * 8 - h * 4) * (uint32_t)sizeof(OpRec);
            half(h, lds32(rec + offsetof(OpRec, base)), false);
#pragma unroll (kStepUnroll)
            for (int cc = 3; cc >= 0; cc--)
                step(rec - (uint32_t)cc * (uint32_t)sizeof(OpRec), g * 8 + h * 4 + cc, cc, false);
        }
    }
#pragma unroll
    for (int k = 0; k < NP; k++) {
        mk[k] = (uint64_t)__double2ull_rz(dmax(prev[k], oth[k]));
        if (MEM && mu[k].over(cap)) mk[k] = kInfeasible;
    }
}

// --------------------------- M = 4, 8 PERTURB: device words (tagged f64)
// Generator revision 3 (oracle/pp_oracle.c or_gen): a flipped op is re-drawn
// as base ⊕ (y mod M).  That makes the devices of a half-group (4 ops) one
// SIMD-within-a-register computation per placement, as in schedule_m2p:
//   f7_c  = [u_c < τ] in bit 7 of byte c     (the byte compare of schedule_m2p)
//   dev   = base ⊕ (y ∧ (f7 >> 7)·(M − 1))   (one SHF, one IMAD, one LOP3;
//                                             base = the image's half-group word)
//   cut   = (dev ⊕ dev of the previous step) + 0x7F… (bit 7 of byte c = [dev_c ≠
//           dev_{c−1}], byte values ≤ 7 so nothing carries across bytes)
// Per step one PRMT widens cut_c to a full-word mask and one PRMT + IMAD turn
// dev_c into the address of free[dev_c]; free[] stays in the warp's shared
// region (schedule_f64's M ≥ 3 state: free[pdev] ← prev every step).  The
// arithmetic is schedule_f64's for M ≥ 3, operation for operation; only the
// devices and cut flags are derived differently, so the results are identical
// (the parity suite runs both).
template <int M, int NP, bool MEM, bool RP = false>
__device__ __forceinline__ void schedule_mpw(uint64_t A, uint64_t B, uint64_t dA, uint32_t hk0, uint64_t (&mk)[NP],
                                             uint32_t ops, uint32_t xr, const uint64_t *__restrict__ mem, uint32_t lane,
                                             uint32_t free_off, uint32_t K8, uint64_t cap, uint32_t khi, uint32_t tau,
                                             uint32_t hgw) {
    static_assert(M == 4 || M == 8, "device words need M = 4 or 8");
    constexpr uint32_t H = 0x80808080u;
    const uint32_t tq = (tau <= 128 ? tau : tau - 128) * 0x01010101u;
    const uint32_t amaj = tau <= 128 ? ~0u : 0u;
    double prev[NP];
    uint32_t dw[NP], cw[NP], dprev[NP], aprev[NP];
    // free[d] of placement k lives at fb + d·NP·256 + k·256 (the k·256 folds
    // into the instructions' immediate offsets)
    const uint32_t fb = lane + free_off * NP;
    uint64_t w[NP], y[NP];
    MemUse<M> mu[NP];
#pragma unroll
    for (int k = 0; k < NP; k++) {
        prev[k] = 0.0;
        dprev[k] = 0;                 // device 0 before the first step (schedule_f64's pdev = 0)
        dw[k] = cw[k] = 0;
        w[k] = y[k] = 0;
        aprev[k] = fb;
#pragma unroll
        for (int d = 0; d < M; d++) std_(fb + d * NP * 256 + k * 256, 0.0);
        if (MEM) mu[k].init();
    }
    uint32_t x = xr;
    auto refresh = [&]() {
#pragma unroll
        for (int k = 0; k < NP; k++) {
            w[k] = mix64(A + (uint64_t)k * dA);
            y[k] = mix64(B + (uint64_t)k * dA);
        }
    };
    auto half = [&](uint32_t h, uint32_t bw, bool fwd) {
#pragma unroll
        for (int k = 0; k < NP; k++) {
            const uint32_t u = h ? (uint32_t)(w[k] >> 32) : (uint32_t)w[k];
            const uint32_t yv = h ? (uint32_t)(y[k] >> 32) : (uint32_t)y[k];
            const uint32_t xx = (u | H) - tq;
            const uint32_t mj = lop3<0xE8>(u, xx, amaj);                        // MAJ: bit 7 = no flip
            const uint32_t f7 = lop3<0x30>(k == 0 ? hk0 : H, mj, 0u);           // hk ∧ ¬mj: bit 7 = flip
            const uint32_t fm = (f7 >> 7) * (uint32_t)(M - 1);                  // M − 1 in flipped bytes
            dw[k] = lop3<0x78>(bw, yv, fm);                                     // base ⊕ (y ∧ fm)
            const uint32_t sh = fwd ? prmt(dw[k], dprev[k], 0x2107u) : prmt(dw[k], dprev[k], 0x4321u);
            cw[k] = (dw[k] ^ sh) + 0x7F7F7F7Fu;                                 // bit 7 of byte c: cut_c
            dprev[k] = dw[k];
        }
    };
    // records are read in address order (forward, then backward): with RP the
    // next step's record is loaded when a step starts (+10 registers; used when
    // few warps are resident, e.g. GNMT: profiles/r02_ab_rec_prefetch.txt)
    double rcost = 0.0, rc0 = 0.0;
    uint4 rb = {0, 0, 0, 0};
    if constexpr (RP) {
        rcost = ldd(ops);
        rc0 = ldd(ops + 8);
        rb = lds128(ops + 16);
    }
    // free[dev] of the next step of the half-group, loaded at the end of the
    // current step (after its write-back of free[pdev]), so the shared-memory
    // latency is off the step's dependency chain.  If the next step stays on
    // the current device the value is that device's stale copy, which no
    // step uses (chain: ≤ prev ≤ t; join: the cut factor 0 selects prev).
    double fn[NP];
    auto step = [&](uint32_t rec, uint32_t p, uint32_t c, bool fwd) {
        const bool pre_in = PP_MPW_PREFETCH && (fwd ? c != 0 : c != 3);    // compile-time (unrolled c)
        const bool pre_out = PP_MPW_PREFETCH && (fwd ? c != 3 : c != 0);
        double cost, c0;
        uint4 b;
        if constexpr (RP) {   // this step's record was loaded when the previous step started
            cost = rcost;
            c0 = rc0;
            b = rb;
            rcost = ldd(rec + sizeof(OpRec));
            rc0 = ldd(rec + sizeof(OpRec) + 8);
            rb = lds128(rec + sizeof(OpRec) + 16);
        } else {
            cost = ldd(rec);
            c0 = ldd(rec + 8);
            b = lds128(rec + 16);
        }
        double cut[NP];
        uint32_t dc[NP], a[NP];
#pragma unroll
        for (int k = 0; k < NP; k++) {
            const uint32_t m = prmt(cw[k], 0u, 0x8888u | (c * 0x1111u));         // all ones iff cut_c
            cut[k] = __hiloint2double((int)(m & khi), 0);                       // 1.0 or 0.0
            dc[k] = prmt(dw[k], 0u, 0x4440u | c);                               // dev_c
            a[k] = dc[k] * (uint32_t)(NP * 256) + fb;                           // &free[dev_c] − k·256
        }
        if (b.z == 0) {
            // chain step: s = max(prev + cut·c0, free[dev]); free[pdev] ← prev
#pragma unroll
            for (int k = 0; k < NP; k++) {
                const double f = pre_in ? fn[k] : ldd(a[k] + k * 256);   // stale (≤ prev ≤ t) unless cut: no cut factor
                std_(aprev[k] + k * 256, prev[k]);
                const double t = __fma_rn(c0, cut[k], prev[k]);
                prev[k] = dmax_add(t, f, cost);
                aprev[k] = a[k];
            }
        } else {
            double r[NP];
            if (b.x == kFromPrev) {
#pragma unroll
                for (int k = 0; k < NP; k++) r[k] = __fma_rn(c0, cut[k], prev[k]);
            } else {
#pragma unroll
                for (int k = 0; k < NP; k++) r[k] = cut_add_f64<M>(ldd(lane + b.x * NP + k * 256), dc[k], c0, khi);
            }
            const uint32_t nx = b.z & 0xFFFFu;
#pragma unroll 1
            for (uint32_t q = 0; q < nx; q++) {   // further inputs (uniform trip count)
                double ce;
                uint32_t ez;
                if (PP_EXTRA_SPLIT) {
                    ce = ldd(x);
                    ez = lds32(x + 8);
                } else {
                    const uint4 e = lds128(x);
                    ce = __hiloint2double((int)e.y, (int)e.x);
                    ez = e.z;
                }
                x += sizeof(ExtraRec);
#pragma unroll
                for (int k = 0; k < NP; k++)
                    r[k] = dmax(r[k], cut_add_f64<M>(ldd(lane + ez * NP + k * 256), dc[k], ce, khi));
            }
#pragma unroll
            for (int k = 0; k < NP; k++) {
                // free[dev] = cut ? free[dev] (shared) : prev, exact on the FP64 pipe
                const double f = __fma_rn(cut[k], __dadd_rn(pre_in ? fn[k] : ldd(a[k] + k * 256), -prev[k]), prev[k]);
                std_(aprev[k] + k * 256, prev[k]);
                prev[k] = dmax_add(clear_tag(r[k]), f, cost);
                aprev[k] = a[k];
            }
        }
        if (b.y != kNoStore) {
#pragma unroll
            for (int k = 0; k < NP; k++) std_(lane + b.y * NP + k * 256, with_tag(prev[k], dc[k]));
        }
        if (pre_out) {
            const uint32_t cn = fwd ? c + 1 : c - 1;
#pragma unroll
            for (int k = 0; k < NP; k++)
                fn[k] = ldd(prmt(dw[k], 0u, 0x4440u | cn) * (uint32_t)(NP * 256) + fb + k * 256);
        }
        if (MEM && fwd) {
            const uint64_t mm = mem[p];
#pragma unroll
            for (int k = 0; k < NP; k++) mu[k].add(dc[k], mm);
        }
    };
    constexpr int kHalfUnroll = NP >= 4 ? 1 : 2;
    const uint32_t G = K8 / 8;
    for (uint32_t g = 0; g < G; g++) {           // forward, π order
        refresh();
        A += kGamma;
        B += kGamma;
#pragma unroll (kHalfUnroll)
        for (uint32_t h = 0; h < 2; h++) {
            const uint32_t rec = ops + (g * 8 + h * 4) * (uint32_t)sizeof(OpRec);
            half(h, lds32(hgw + 4 * (2 * g + h)), true);
#pragma unroll
            for (uint32_t cc = 0; cc < 4; cc++) step(rec + cc * (uint32_t)sizeof(OpRec), g * 8 + h * 4 + cc, cc, true);
        }
    }
#pragma unroll
    for (int k = 0; k < NP; k++) dprev[k] >>= 24;   // byte 0 := the device of the last forward step
    for (uint32_t g = G; g-- > 0;) {             // backward, reverse π order
        A -= kGamma;
        B -= kGamma;
        refresh();
#pragma unroll (kHalfUnroll)
        for (uint32_t h = 2; h-- > 0;) {
            const uint32_t rec = ops + (2 * K8 - 1 - g * 8 - h * 4) * (uint32_t)sizeof(OpRec);
            half(h, lds32(hgw + 4 * (2 * g + h)), false);
#pragma unroll
            for (int cc = 3; cc >= 0; cc--)
                step(rec - (uint32_t)cc * (uint32_t)sizeof(OpRec), g * 8 + h * 4 + cc, cc, false);
        }
    }
#pragma unroll
    for (int k = 0; k < NP; k++) {
        std_(aprev[k] + k * 256, prev[k]);
        double v = 0.0;
#pragma unroll
        for (int d = 0; d < M; d++) v = dmax(v, ldd(fb + d * NP * 256 + k * 256));
        mk[k] = (uint64_t)__double2ull_rz(v);
        if (MEM && mu[k].over(cap)) mk[k] = kInfeasible;
    }
}

#ifndef PP_MPW
#define PP_MPW 1   // the device-word schedule for M = 4, 8 PERTURB (0: schedule_f64, for A/B)
#endif

#ifndef PP_M2P
#define PP_M2P 1   // the cut-word schedule for M = 2 PERTURB (0: schedule_f64, for A/B)
#endif

template <int M, int NP, bool MEM, bool F64, bool HW, class Gen>
__device__ __forceinline__ void schedule_np(Gen &gen, uint64_t (&mk)[NP], uint32_t ops, uint32_t xr,
                                            const uint64_t *__restrict__ mem, uint32_t lane, uint32_t free_off,
                                            uint32_t K8, uint64_t cap, uint32_t khi, uint32_t cls, uint32_t tau,
                                            uint32_t hq = 0, uint32_t nslot = 0) {
    if constexpr (F64 && M >= 2)
        schedule_f64<M, NP, MEM, HW>(gen, mk, ops, xr, mem, lane, free_off, K8, cap, khi, cls, hq, nslot);
    else schedule_gen<M, NP, MEM, F64>(gen, mk, ops, xr, mem, lane, free_off, K8, cap);
}

__device__ __forceinline__ bool lex_less(uint64_t m1, uint64_t i1, uint64_t m2, uint64_t i2) {
    return m1 < m2 || (m1 == m2 && i1 < i2);
}

// ---- argmin epilogue: warp shuffle → CTA (shared) → grid (the last CTA to
// finish reduces the per-CTA partials and resets the ticket and tile counter)
__device__ __forceinline__ void grid_argmin(const KParams &P, uint64_t best_mk, uint64_t best_i, uint64_t *red_mk,
                                            uint64_t *red_i, bool &is_last) {
    const uint32_t tid = threadIdx.x;
    const uint32_t lane = tid & 31, warp = tid >> 5;
    const uint32_t nthreads = blockDim.x;
    const uint32_t wpb = nthreads >> 5;
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
        *P.g_tile = 0;
    }
}

// ------------------------------------------------------------------ kernel
template <int M, int GEN, bool MEM, bool WRITE_ALL, bool F64, int NP, bool HW, bool RP = false>
__global__ void __launch_bounds__(PP_CTA_THREADS, PP_MIN_CTAS) search_kernel(const KParams P) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint64_t red_mk[32], red_i[32];
    __shared__ bool is_last;

    const uint32_t tid = threadIdx.x;
    const uint32_t lane = tid & 31, warp = tid >> 5;
    const uint32_t nthreads = blockDim.x;

    // ---- stage the image with bulk TMA copies completing on one mbarrier
    const uint32_t mbar_addr = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_addr));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar_addr), "r"(P.image_bytes)
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
    }
    // this lane's state; the always-zero slot is never written again
    const uint32_t smem_base = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t lane_region = smem_base + P.smem_slots_off + warp * P.region_bytes + lane * 8;
#pragma unroll
    for (int k = 0; k < NP; k++) sts64(lane_region + P.zero_off * NP + k * 256, 0);
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

    const uint32_t ops = smem_base;
    const uint32_t xr = smem_base + P.off_extra;
    const uint64_t *mem = reinterpret_cast<const uint64_t *>(smem + P.off_mem);
    const uint32_t *orig = reinterpret_cast<const uint32_t *>(smem + P.off_orig);

    uint64_t best_mk = kInfeasible, best_i = kInfeasible;
    bool have = false;
    const uint64_t n = P.end - P.begin;
    constexpr uint32_t TILE = 32 * NP;
    constexpr bool kM2P = PP_M2P && F64 && M == 2 && !HW;   // schedule_m2p
    constexpr bool kMPW = PP_MPW && F64 && (M == 4 || M == 8) && !HW;   // schedule_mpw
    // GEN_SYM: a unit is a task (one RGS prefix × a block of NP last-position
    // values), one per lane, so a tile is 32 tasks
    const uint64_t ntiles = (n + (GEN == GEN_SYM ? 31 : TILE - 1)) / (GEN == GEN_SYM ? 32 : TILE);
    const uint64_t wpb = nthreads >> 5;
    // Tile schedule: the argmin kernels take tiles from a global counter (reset
    // by the last CTA), so a warp that runs ahead takes more and none idles at
    // the closing barrier while others still hold a static share (GNMT M = 2:
    // +13%, BigLSTM +1.5%, Inception −0.9%; profiles/r02_ab_tiles.txt).  The
    // write-all kernels stride statically.  PP_TILE_PREFETCH claims the next
    // tile when a tile starts (A/B).
    constexpr bool kDyn = !WRITE_ALL && PP_DYN_TILES;
    auto claim = [&]() -> uint64_t {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(P.g_tile, 1ull);
        return (uint64_t)__shfl_sync(0xffffffffu, v, 0);
    };
    uint64_t tile = kDyn ? claim() : blockIdx.x * wpb + warp;
    while (tile < ntiles) {
        unsigned long long pre = 0;
        if (kDyn && PP_TILE_PREFETCH && lane == 0) pre = atomicAdd(P.g_tile, 1ull);
        uint64_t off[NP], idx[NP];
        bool valid[NP];
#pragma unroll
        for (int k = 0; k < NP; k++) {
            off[k] = tile * (GEN == GEN_SYM ? 32 : TILE) + (GEN == GEN_SYM ? lane : k * 32 + lane);
            valid[k] = off[k] < n;
            idx[k] = P.begin + (valid[k] ? off[k] : n - 1);
        }
        // the generators' lane placements i_0 + 32k (unclamped: results of
        // lanes past the end are discarded); only i_0 can be candidate 0
        const uint64_t i0 = P.begin + tile * TILE + lane;
        uint64_t mk[NP];
        if constexpr (GEN == GEN_SYM) {
            // task t = (prefix rank) · B + block: the lane's placements are the
            // RGS prefix of π positions 0..K−2 followed by the values
            // v = block·NP + k at position K−1 (valid iff v < min(m + 1, M),
            // m = devices the prefix uses).  They share the forward prefix:
            // ⌊(K−1)/4⌋ half-groups run for placement 0 only (schedule_f64).
            constexpr uint32_t B = (M + NP - 1) / NP;
            constexpr uint32_t b = Bits<M>::b, PF = b ? 64 / b : 64;
            RgsGen<M, NP> g;
            uint64_t plo, phi;
            const uint32_t m = RgsGen<M, NP>::unrank(idx[0] / B, P.K - 1, P.g_rgs, plo, phi);
            const uint32_t blk = (uint32_t)(idx[0] % B);
            const uint32_t j = P.K - 1;
#pragma unroll
            for (int k = 0; k < NP; k++) {
                const uint32_t v = blk * NP + (uint32_t)k;
                const bool ok = v < min(m + 1, (uint32_t)M);
                valid[k] = valid[k] && ok;
                const uint64_t f = (uint64_t)(ok ? v : 0u);
                g.lo[k] = plo | (j < PF ? f << (j * b) : 0ull);
                g.hi[k] = phi | (j < PF ? 0ull : f << ((j - PF) * b));
            }
            schedule_np<M, NP, MEM, F64, HW>(g, mk, ops, xr, mem, lane_region, P.free_off, P.K8, P.cap, P.one_hi,
                                              smem_base + P.off_cls, P.tau, (P.K - 1) / 4, P.zero_off / kSlotUnit);
            // the class's index is its smallest Gray index, needed only when
            // the class can still win
#pragma unroll
            for (int k = 0; k < NP; k++)
                idx[k] = (valid[k] && mk[k] <= best_mk) ? gray_min_index<M>(g.lo[k], g.hi[k], P.K) : kInfeasible;
        } else if (GEN == GEN_GRAY) {
            GrayGen<M, NP> g;
            g.init(idx, P.K);
            schedule_np<M, NP, MEM, F64, HW>(g, mk, ops, xr, mem, lane_region, P.free_off, P.K8, P.cap, P.one_hi,
                                              smem_base + P.off_cls, P.tau);
        } else if (GEN == GEN_RANDOM) {
            RandomGen<M, NP> g;
            g.init(i0, P.seed, P.K);
            schedule_np<M, NP, MEM, F64, HW>(g, mk, ops, xr, mem, lane_region, P.free_off, P.K8, P.cap, P.one_hi,
                                              smem_base + P.off_cls, P.tau);
        } else if constexpr (GEN == GEN_PERTURB && kM2P) {
            const uint64_t Wd = (P.K + 7) / 8;
            const uint64_t A = (P.seed ^ 0xD1B54A32D192ED03ull) + kGamma * (i0 * Wd + 1);
            schedule_m2p<NP, MEM, RP>(A, kGamma * 32ull * Wd, i0 == 0 ? 0u : 0x80808080u, mk, ops, xr, mem, lane_region,
                                  P.K8, P.cap, P.one_hi, P.tau);
        } else if constexpr (GEN == GEN_PERTURB && kMPW) {
            const uint64_t Wd = (P.K + 7) / 8;
            const uint64_t A = (P.seed ^ 0xD1B54A32D192ED03ull) + kGamma * (i0 * Wd + 1);
            const uint64_t B = (P.seed ^ 0x8CB92BA72F3D8DD7ull) + kGamma * (i0 * Wd + 1);
            schedule_mpw<M, NP, MEM, RP>(A, B, kGamma * 32ull * Wd, i0 == 0 ? 0u : 0x80808080u, mk, ops, xr, mem,
                                     lane_region, P.free_off, P.K8, P.cap, P.one_hi, P.tau, smem_base + P.off_hgw);
        } else if (GEN == GEN_PERTURB) {
            PerturbGen<M, NP> g;
            g.init(i0, P.seed, P.K, P.tau);
            schedule_np<M, NP, MEM, F64, HW>(g, mk, ops, xr, mem, lane_region, P.free_off, P.K8, P.cap, P.one_hi,
                                              smem_base + P.off_cls, P.tau);
        } else {
            ExplicitGen<M, NP> g;
#pragma unroll
            for (int k = 0; k < NP; k++) {
                g.row[k] = P.g_place + (idx[k] - P.begin) * (uint64_t)P.K;
                g.bad[k] = 0;
            }
            g.orig = orig;
            schedule_np<M, NP, MEM, F64, HW>(g, mk, ops, xr, mem, lane_region, P.free_off, P.K8, P.cap, P.one_hi,
                                              smem_base + P.off_cls, P.tau);
#pragma unroll
            for (int k = 0; k < NP; k++)
                if (g.bad[k]) mk[k] = kInfeasible;
        }
#pragma unroll
        for (int k = 0; k < NP; k++) {
            if (WRITE_ALL) {
                if (valid[k]) P.g_makespan[off[k]] = mk[k];
            } else if (valid[k] && (!have || lex_less(mk[k], idx[k], best_mk, best_i))) {
                best_mk = mk[k];
                best_i = idx[k];
                have = true;
            }
        }
        if (!kDyn) tile += (uint64_t)gridDim.x * wpb;
        else if (PP_TILE_PREFETCH) tile = (uint64_t)__shfl_sync(0xffffffffu, pre, 0);
        else tile = claim();
    }
    if (WRITE_ALL) return;

    grid_argmin(P, best_mk, best_i, red_mk, red_i, is_last);
}

// ------------------------------------------------- global-state tier
// the schedule body of the global tier: schedule_f64 when the image is
// f64-encoded (time bound < 2^49 ps) and M ≥ 2, else schedule_gen
// placements per lane on the global tier: big_np(M) (internal.h; A/B in
// profiles/r02_big_bench_np.txt: NP = 2 is faster at M ≤ 2, NP = 1 at M ≥ 3,
// where NP = 2 needs 122–128 registers and halves the resident warps)
template <int M, bool F64, int NP, class Gen>
__device__ __forceinline__ void big_schedule(Gen &g, uint64_t (&mk)[NP], uint64_t ops, uint64_t xr,
                                             const uint64_t *__restrict__ mem, uint64_t lane, const KParams &P,
                                             uint64_t cap) {
    if constexpr (F64 && M >= 2)
        schedule_f64<M, NP, true, false, Gen, GmemSpace>(g, mk, ops, xr, mem, lane, P.free_off, P.K8, cap, P.one_hi,
                                                         0);
    else
        schedule_gen<M, NP, true, F64, Gen, GmemSpace>(g, mk, ops, xr, mem, lane, P.free_off, P.K8, cap);
}

template <int M, int GEN, bool F64>
__global__ void __launch_bounds__(256) search_big_kernel(const KParams P) {
    constexpr int NP = big_np(M);
    constexpr uint32_t TILE = 32 * NP;
    __shared__ uint64_t red_mk[32], red_i[32];
    __shared__ bool is_last;
    const uint32_t tid = threadIdx.x;
    const uint32_t lane = tid & 31, warp = tid >> 5;
    const uint64_t wpb = blockDim.x >> 5;
    const bool write_all = P.g_makespan != nullptr;
    const uint64_t cap = P.cap ? P.cap : ~0ull;
    const uint64_t ops = reinterpret_cast<uint64_t>(P.g_image);
    const uint64_t xr = ops + P.off_extra;
    const uint64_t *mem = reinterpret_cast<const uint64_t *>(P.g_image + P.off_mem);
    const uint32_t *orig = reinterpret_cast<const uint32_t *>(P.g_image + P.off_orig);
    const uint64_t lane_region =
        reinterpret_cast<uint64_t>(P.g_state) + (blockIdx.x * wpb + warp) * (uint64_t)P.region_bytes + lane * 8u;
#pragma unroll
    for (int k = 0; k < NP; k++)   // the always-zero slot
        *reinterpret_cast<uint64_t *>(lane_region + P.zero_off * NP + k * 256) = 0;

    uint64_t best_mk = kInfeasible, best_i = kInfeasible;
    const uint64_t n = P.end - P.begin;
    const uint64_t ntiles = (n + TILE - 1) / TILE;
    auto claim = [&]() -> uint64_t {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(P.g_tile, 1ull);
        return (uint64_t)__shfl_sync(0xffffffffu, v, 0);
    };
    uint64_t tile = write_all ? blockIdx.x * wpb + warp : claim();
    while (tile < ntiles) {
        // the lane's placements i_0 + 32k (search_kernel's layout)
        uint64_t off[NP], idx[NP];
        bool valid[NP];
#pragma unroll
        for (int k = 0; k < NP; k++) {
            off[k] = tile * TILE + k * 32 + lane;
            valid[k] = off[k] < n;
            idx[k] = P.begin + (valid[k] ? off[k] : n - 1);
        }
        const uint64_t i0 = P.begin + tile * TILE + lane;
        uint64_t mk[NP];
        if constexpr (GEN == GEN_GRAY) {
            GrayGen<M, NP> g;
            g.init(idx, P.K);
            big_schedule<M, F64, NP>(g, mk, ops, xr, mem, lane_region, P, cap);
        } else if constexpr (GEN == GEN_RANDOM) {
            RandomGen<M, NP> g;
            g.init(i0, P.seed, P.K);
            big_schedule<M, F64, NP>(g, mk, ops, xr, mem, lane_region, P, cap);
        } else if constexpr (GEN == GEN_PERTURB) {
            PerturbGen<M, NP> g;
            g.init(i0, P.seed, P.K, P.tau);
            big_schedule<M, F64, NP>(g, mk, ops, xr, mem, lane_region, P, cap);
        } else {
            ExplicitGen<M, NP> g;
#pragma unroll
            for (int k = 0; k < NP; k++) {
                g.row[k] = P.g_place + (idx[k] - P.begin) * (uint64_t)P.K;
                g.bad[k] = 0;
            }
            g.orig = orig;
            big_schedule<M, F64, NP>(g, mk, ops, xr, mem, lane_region, P, cap);
#pragma unroll
            for (int k = 0; k < NP; k++)
                if (g.bad[k]) mk[k] = kInfeasible;
        }
#pragma unroll
        for (int k = 0; k < NP; k++) {
            if (write_all) {
                if (valid[k]) P.g_makespan[off[k]] = mk[k];
            } else if (valid[k] && lex_less(mk[k], idx[k], best_mk, best_i)) {
                best_mk = mk[k];
                best_i = idx[k];
            }
        }
        tile = write_all ? tile + (uint64_t)gridDim.x * wpb : claim();
    }
    if (write_all) return;
    grid_argmin(P, best_mk, best_i, red_mk, red_i, is_last);
}
template <int M, int GEN, bool F64>
int launch_search_big(const KParams &p, int grid, int threads, int smem, void *stream) {
    search_big_kernel<M, GEN, F64><<<grid, threads, smem, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------- round update
// One CTA.  Reads the round winner (makespan, index) — the local argmin on one
// GPU, or the NCCL-reduced key/index on several — regenerates its placement,
// keeps the overall best (first round reaching the minimum) and moves the
// PERTURB base to the winner (candidate 0 is the base, so the winner differs
// from the base only when it is strictly better), patching
// the new base into the op records of the device image.
template <int M, int GEN>
__global__ void __launch_bounds__(256) round_update_kernel(const UParams U) {
    __shared__ uint64_t mk_s, idx_s;
    __shared__ int improve;
    uint64_t *s = U.s;
    __shared__ int move;
    if (threadIdx.x == 0) {
        uint64_t mk, idx;
        if (U.multi) {   // the exchanged winner (protocol.h)
            mk = proto::key_makespan(s[SC_KEY_GLOBAL]);
            idx = s[SC_IDX_GLOBAL];
        } else {
            mk = s[SC_LOCAL_MK];
            idx = s[SC_LOCAL_IDX];
        }
        mk_s = mk;
        idx_s = idx;
        improve = idx != proto::kNone && ((U.round == 0) || (mk < s[SC_BEST_MK]));
        move = proto::moves_base(idx);
    }
    __syncthreads();
    if (idx_s == proto::kNone) return;   // no candidate anywhere (cannot happen for count ≥ 1)
    const uint64_t ii[1] = {idx_s};
    for (uint32_t p = threadIdx.x; p < U.K; p += blockDim.x) {
        uint32_t d;
        if (GEN == GEN_GRAY) {
            GrayGen<M, 1> g;
            g.init(ii, U.K);
            d = g.dev(0, p, p % 8, 0);
        } else if (GEN == GEN_RANDOM) {
            RandomGen<M, 1> g;
            g.init(idx_s, U.seed, U.K);
            g.refresh(p / 8);
            g.sub((p / 4) & 1);
            d = g.dev(0, p, p % 4, 0);
        } else {
            PerturbGen<M, 1> g;
            g.init(idx_s, U.seed, U.K, U.tau);
            g.refresh(p / 8);
            g.sub((p / 4) & 1);
            d = g.dev(0, p, p % 4, U.base[p]);
        }
        U.winner[p] = (uint8_t)Dev<M>::canon(d);
    }
    __syncthreads();
    OpRec *ops = reinterpret_cast<OpRec *>(U.image);
    uint32_t *hgw = reinterpret_cast<uint32_t *>(U.image + U.off_hgw);
    for (uint32_t p = threadIdx.x; p < U.K8; p += blockDim.x) {
        const uint8_t d = p < U.K ? U.winner[p] : 0;
        if (GEN == GEN_PERTURB && move) {
            const uint32_t w = half_group_word(U.winner, p, U.K);
            if (p < U.K) U.base[p] = d;
            ops[p].base = d | w;
            ops[2 * U.K8 - 1 - p].base = d | w;
            if ((p & 3) == 0) hgw[p / 4] = half_group_bytes(U.winner, p / 4, U.K);
        }
        if (improve && p < U.K) U.best_place[p] = d;
    }
    if (threadIdx.x == 0 && improve) {
        s[SC_BEST_MK] = mk_s;
        s[SC_BEST_IDX] = idx_s;
        s[SC_BEST_ROUND] = U.round;
    }
}

template <int M, int GEN, bool MEM, bool WRITE_ALL, bool F64, int NP, bool HW, bool RP = false>
int launch_search(const KParams &p, int grid, int threads, int smem, void *stream) {
    search_kernel<M, GEN, MEM, WRITE_ALL, F64, NP, HW, RP><<<grid, threads, smem, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

template <int M, int GEN>
int launch_update(const UParams &u, void *stream) {
    round_update_kernel<M, GEN><<<1, 256, 0, (cudaStream_t)stream>>>(u);
    return (int)cudaGetLastError();
}

}  // namespace pp
