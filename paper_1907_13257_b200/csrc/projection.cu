// projection.cu — end-to-end projection cells and the DP→hybrid crossover on
// the GPU, exact in unsigned 128-bit integers.
//
// Cell (M, N)  (SURVEY.md §8(c) O8–O10; readings R10–R15):
//   W = N/M (M ∤ N ⇒ infeasible), G = W·B
//   E = E(G): knot value, or ⌊linear interpolation in G⌋; outside ⇒ infeasible
//   AR(W) = 0 (W = 1 or tier BW = 0) else ⌈2(W−1)·S·10^12/(W·BW)⌉ + 2(W−1)·α,
//           tier = intra iff N ≤ node_size
//   T = ⌊(T_1 + AR)·T_M / T_1⌋ (EQ5 = SU^M·SE_W, Eq. 5)
//       or T_M + AR (TIME)
//   NEXT f4: accumulation factors a (G = W·B·a, T = ⌊(a·T_1 + AR)·T_M/T_1⌋ or
//   a·T_M + AR, the least-C a kept) and per-device shards (AR = max_d AR(S_d))
//   steps = ⌈D/G⌉, C = T·steps·E (Eq. 1)
// Crossover (Eq. 6, strict; R16).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.h"

namespace pp {

typedef unsigned __int128 u128;

constexpr int kMaxKnots = 64;
constexpr int kMaxAccum = 32;

struct ProjParams {
    uint64_t D, grad, bw_in, lat_in, bw_out, lat_out, t1;
    uint32_t B, n_knots, node, mode;
    uint32_t nM, N_max, nA, sharded;
    uint32_t Ms[8];
    uint64_t TM[8];
    uint64_t kG[kMaxKnots], kE[kMaxKnots];
    uint32_t A[kMaxAccum];           // accumulation factors (NEXT f4)
    uint64_t shard[8][8];            // per-M per-device gradient shards
};

__device__ __forceinline__ int bitlen(u128 x) {
    uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
    return hi ? 128 - __clzll((long long)hi) : (lo ? 64 - __clzll((long long)lo) : 0);
}

// ring all-reduce of S bytes over W workers in the tier of N devices
__device__ int ring_ar(const ProjParams &P, uint64_t W, uint32_t N, uint64_t S, u128 &A) {
    A = 0;
    if (W <= 1) return 0;
    const bool intra = N <= P.node;
    const uint64_t bw = intra ? P.bw_in : P.bw_out;
    const uint64_t al = intra ? P.lat_in : P.lat_out;
    if (!bw) return 0;
    const u128 steps2 = (u128)2 * (W - 1);
    if (bitlen(steps2) + bitlen(S) + 40 > 127) return -3;
    const u128 num = steps2 * S * (u128)1000000000000ull;
    const u128 den = (u128)W * bw;
    A = num / den + ((num % den) ? 1 : 0) + steps2 * al;
    return 0;
}

// E(G) from the knots; false outside them
__device__ bool epochs_of(const ProjParams &P, uint64_t g, uint64_t &E) {
    if (g < P.kG[0] || g > P.kG[P.n_knots - 1]) return false;
    for (uint32_t i = 0; i < P.n_knots; i++) {
        if (P.kG[i] == g) { E = P.kE[i]; return true; }
        if (i + 1 < P.n_knots && P.kG[i] < g && g < P.kG[i + 1]) {
            u128 num = (u128)P.kE[i] * (P.kG[i + 1] - g) + (u128)P.kE[i + 1] * (g - P.kG[i]);
            E = (uint64_t)(num / (P.kG[i + 1] - P.kG[i]));
            return true;
        }
    }
    return false;
}

// returns 0 = ok (infeasible cells have feasible = 0), -3 = range
__device__ int cell_value(const ProjParams &P, uint32_t m, uint32_t N, pp_cell &c) {
    const uint32_t M = P.Ms[m];
    const uint64_t TM = P.TM[m];
    c = pp_cell{0, 0, 0, 0, 0, 0, 0};
    if (N % M) return 0;
    const uint64_t W = N / M;
    u128 A = 0;
    if (P.sharded) {   // placement-aware: the slowest device's shard (R24)
        for (uint32_t d = 0; d < M && d < 8; d++) {
            u128 Ad;
            if (ring_ar(P, W, N, P.shard[m][d], Ad)) return -3;
            A = Ad > A ? Ad : A;
        }
    } else if (ring_ar(P, W, N, P.grad, A)) {
        return -3;
    }
    u128 best = 0;
    for (uint32_t j = 0; j < P.nA; j++) {
        const uint64_t a = P.A[j];
        const u128 G = (u128)W * P.B * a;
        if (G >> 64) continue;
        const uint64_t g = (uint64_t)G;
        uint64_t E;
        if (!epochs_of(P, g, E)) continue;
        u128 T;
        if (P.mode == 0) {
            const u128 x = (u128)a * P.t1 + A;
            if (bitlen(x) + bitlen(TM) > 127) return -3;
            T = x * TM / P.t1;
        } else {
            T = (u128)a * TM + A;
        }
        if (T >> 64) return -3;
        const uint64_t steps = (P.D + g - 1) / g;
        if (bitlen(T) + bitlen(steps) + bitlen(E) > 127) return -3;
        const u128 C = T * steps * E;
        if (!c.feasible || C < best) {
            best = C;
            c.C_lo = (uint64_t)C;
            c.C_hi = (uint64_t)(C >> 64);
            c.step_ps = (uint64_t)T;
            c.steps = steps;
            c.uepochs = E;
            c.feasible = 1;
            c.accum = (uint32_t)a;
        }
    }
    return 0;
}

__global__ void project_kernel(const ProjParams P, pp_cell *cells, int *err) {
    const uint32_t total = P.nM * P.N_max;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const uint32_t m = t / P.N_max, N = t % P.N_max + 1;
        pp_cell c;
        int rc = cell_value(P, m, N, c);
        if (rc) atomicMin(err, rc);
        cells[t] = c;
    }
}

__device__ __forceinline__ u128 cellC(const pp_cell &c) { return ((u128)c.C_hi << 64) | c.C_lo; }

struct CrossParams {
    uint32_t nM, N_max, m1;
    uint32_t Ms[8];
};

// One CTA.  Thread t owns the contiguous chunk of N values [t·L, (t+1)·L).
__global__ void __launch_bounds__(1024) crossover_kernel(const CrossParams X, const pp_cell *cells,
                                                         pp_crossover_result *out, uint32_t *best_m) {
    __shared__ unsigned nstar_m[8];
    __shared__ unsigned viol_m[8];
    __shared__ u128 chunk_min[1024];
    __shared__ unsigned vs_best;
    const uint32_t nt = blockDim.x, t = threadIdx.x;
    const uint32_t NM = X.N_max;
    const uint32_t L = (NM + nt - 1) / nt;
    const uint32_t lo = t * L + 1, hi = min(NM, (t + 1) * L);   // N in [lo, hi]
    const pp_cell *dp = cells + (size_t)X.m1 * NM;
    if (t < 8) { nstar_m[t] = 0xFFFFFFFFu; viol_m[t] = 0xFFFFFFFFu; }
    if (t == 0) vs_best = 0xFFFFFFFFu;
    __syncthreads();

    // n_star_M: first N with both feasible and C(M,N) < C(1,N)
    for (uint32_t m = 0; m < X.nM; m++) {
        if (m == X.m1) continue;
        const pp_cell *hy = cells + (size_t)m * NM;
        for (uint32_t N = lo; N <= hi; N++) {
            const pp_cell &a = hy[N - 1], &b = dp[N - 1];
            if (a.feasible && b.feasible && cellC(a) < cellC(b)) { atomicMin(&nstar_m[m], N); break; }
        }
    }
    __syncthreads();
    // persistence: any N ≥ n_star_M where both are feasible and hybrid is not better
    for (uint32_t m = 0; m < X.nM; m++) {
        if (m == X.m1 || nstar_m[m] == 0xFFFFFFFFu) continue;
        const pp_cell *hy = cells + (size_t)m * NM;
        for (uint32_t N = max(lo, nstar_m[m]); N <= hi; N++) {
            const pp_cell &a = hy[N - 1], &b = dp[N - 1];
            if (a.feasible && b.feasible && !(cellC(a) < cellC(b))) { atomicMin(&viol_m[m], N); break; }
        }
    }
    // best M per N, and the chunk's minimum feasible DP value (for the prefix min)
    const u128 kNone = ~(u128)0;
    u128 cm = kNone;
    for (uint32_t N = lo; N <= hi; N++) {
        int bm = -1;
        u128 bv = 0;
        for (uint32_t m = 0; m < X.nM; m++) {
            const pp_cell &a = cells[(size_t)m * NM + N - 1];
            if (!a.feasible) continue;
            const u128 v = cellC(a);
            if (bm < 0 || v < bv || (v == bv && X.Ms[m] < X.Ms[bm])) { bm = (int)m; bv = v; }
        }
        if (best_m) best_m[N - 1] = bm < 0 ? 0u : X.Ms[bm];
        if (dp[N - 1].feasible && cellC(dp[N - 1]) < cm) cm = cellC(dp[N - 1]);
    }
    chunk_min[t] = cm;
    __syncthreads();
    // inclusive prefix-min over chunks (Hillis–Steele)
    for (uint32_t o = 1; o < nt; o <<= 1) {
        u128 v = (t >= o) ? chunk_min[t - o] : kNone;
        __syncthreads();
        if (v < chunk_min[t]) chunk_min[t] = v;
        __syncthreads();
    }
    // walk the chunk with the running min of C(1, N') over N' ≤ N
    u128 run = (t > 0) ? chunk_min[t - 1] : kNone;
    for (uint32_t N = lo; N <= hi; N++) {
        if (dp[N - 1].feasible && cellC(dp[N - 1]) < run) run = cellC(dp[N - 1]);
        if (run == kNone) continue;   // no feasible DP cell at or below N
        bool hit = false;
        for (uint32_t m = 0; m < X.nM; m++) {
            const pp_cell &a = cells[(size_t)m * NM + N - 1];
            if (a.feasible && cellC(a) < run) hit = true;
        }
        if (hit) { atomicMin(&vs_best, N); break; }
    }
    __syncthreads();
    if (t == 0) {
        pp_crossover_result r;
        for (int i = 0; i < 8; i++) { r.n_star_M[i] = 0; r.persistent_M[i] = 0; }
        r.n_star = 0;
        r.m_at_n_star = 0;
        for (uint32_t m = 0; m < X.nM; m++) {
            if (m == X.m1 || nstar_m[m] == 0xFFFFFFFFu) continue;
            r.n_star_M[m] = nstar_m[m];
            r.persistent_M[m] = viol_m[m] == 0xFFFFFFFFu;
            if (r.n_star == 0 || nstar_m[m] < r.n_star) r.n_star = nstar_m[m];
        }
        if (r.n_star) {
            const uint32_t N = r.n_star;
            int bm = -1;
            u128 bv = 0;
            for (uint32_t m = 0; m < X.nM; m++) {
                const pp_cell &a = cells[(size_t)m * NM + N - 1];
                if (!a.feasible) continue;
                const u128 v = cellC(a);
                if (bm < 0 || v < bv || (v == bv && X.Ms[m] < X.Ms[bm])) { bm = (int)m; bv = v; }
            }
            r.m_at_n_star = X.Ms[bm];
        }
        r.n_star_vs_best_dp = vs_best == 0xFFFFFFFFu ? 0 : vs_best;
        *out = r;
    }
}

int launch_project(const ProjParams &P, pp_cell *cells, int *err, void *stream) {
    const uint32_t total = P.nM * P.N_max;
    const int threads = 256;
    const int grid = (int)((total + threads - 1) / threads);
    project_kernel<<<grid, threads, 0, (cudaStream_t)stream>>>(P, cells, err);
    return (int)cudaGetLastError();
}

int launch_crossover(const CrossParams &X, const pp_cell *cells, pp_crossover_result *out, uint32_t *best_m,
                     void *stream) {
    crossover_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(X, cells, out, best_m);
    return (int)cudaGetLastError();
}

// --- tiny helpers of the multi-GPU exchange (stream-ordered, no host sync)
// the two device steps of the round exchange (protocol.h)
__global__ void pack_key_kernel(uint64_t *s, int rank) {
    s[SC_KEY_LOCAL] = proto::key(s[SC_LOCAL_MK], s[SC_LOCAL_IDX], rank);
}
__global__ void contrib_kernel(uint64_t *s) {
    s[SC_IDX_LOCAL] = proto::contrib(s[SC_KEY_GLOBAL], s[SC_KEY_LOCAL], s[SC_LOCAL_IDX]);
}
// Copies a π-order base into the canonical buffer and into OpRec.base of the
// forward and backward records of every position p < K8 (PERTURB): the op's
// device plus the packed half-group word (internal.h, OpRec.base).
__global__ void patch_base_kernel(uint8_t *image, uint8_t *base, const uint8_t *src, uint32_t K, uint32_t K8,
                                  uint32_t off_hgw) {
    OpRec *ops = reinterpret_cast<OpRec *>(image);
    uint32_t *hgw = reinterpret_cast<uint32_t *>(image + off_hgw);
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < K8; p += gridDim.x * blockDim.x) {
        const uint8_t d = p < K ? src[p] : 0;
        if (p < K) base[p] = d;
        const uint32_t w = half_group_word(src, p, K);
        ops[p].base = d | w;
        ops[2 * K8 - 1 - p].base = d | w;
        if ((p & 3) == 0) hgw[p / 4] = half_group_bytes(src, p / 4, K);
    }
}
int launch_patch_base(uint8_t *image, uint8_t *base, const uint8_t *src, uint32_t K, uint32_t K8, uint32_t off_hgw,
                      void *stream) {
    patch_base_kernel<<<(K8 + 255) / 256, 256, 0, (cudaStream_t)stream>>>(image, base, src, K, K8, off_hgw);
    return (int)cudaGetLastError();
}
int launch_pack_key(uint64_t *s, int rank, void *stream) {
    pack_key_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(s, rank);
    return (int)cudaGetLastError();
}
__global__ void unpack_best_kernel(const uint64_t *s, uint64_t *out) {
    out[0] = proto::key_makespan(s[SC_KEY_GLOBAL]);
    out[1] = s[SC_IDX_GLOBAL];
}
int launch_unpack_best(const uint64_t *s, uint64_t *out, void *stream) {
    unpack_best_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(s, out);
    return (int)cudaGetLastError();
}
int launch_contrib(uint64_t *s, void *stream) {
    contrib_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(s);
    return (int)cudaGetLastError();
}

}  // namespace pp

// ------------------------------------------------------------ C ABI (host)
namespace pp {

static int proj_fail(int code, const char *msg) {
    set_error(msg);
    return code;
}

static int bitlen_h(u128 x) {
    int n = 0;
    while (x) { n++; x >>= 1; }
    return n;
}

// Per-call scratch for the error flag and the crossover result.  Both calls
// synchronise their stream before returning, so a call holds its scratch slot
// (a 256-byte device buffer) exactly for its lifetime: it takes a free slot
// of the current device on entry and gives it back on exit (after a stream
// synchronize on an error path).  Concurrent calls on different streams or
// threads therefore never share a buffer (pp.h: distinct calls are
// independent), and after the first call no allocation happens on the path
// (cudaMallocAsync from the default pool re-maps memory after every
// synchronize: ≈0.6 ms per call on B200).
struct ScratchSlot {
    void *p = nullptr;
    int dev = -1;
    cudaStream_t st;
    bool synced = false;
    static std::mutex &mu() {
        static std::mutex m;
        return m;
    }
    static std::vector<std::pair<int, void *>> &pool() {
        static std::vector<std::pair<int, void *>> v;
        return v;
    }
    explicit ScratchSlot(cudaStream_t s) : st(s) {}
    cudaError_t take() {
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        {
            std::lock_guard<std::mutex> lk(mu());
            auto &v = pool();
            for (size_t i = 0; i < v.size(); i++)
                if (v[i].first == dev) {
                    p = v[i].second;
                    v.erase(v.begin() + (long)i);
                    return cudaSuccess;
                }
        }
        return cudaMalloc(&p, 256);
    }
    ~ScratchSlot() {
        if (!p) return;
        if (!synced) cudaStreamSynchronize(st);
        std::lock_guard<std::mutex> lk(mu());
        pool().emplace_back(dev, p);
    }
};

}  // namespace pp

extern "C" int pp_project_e2e(const pp_scenario *sc, int nM, const uint32_t *Ms, const uint64_t *T_M_ps,
                              uint32_t N_max, pp_cell *d_cells, void *stream) {
    using namespace pp;
    if (!sc || !Ms || !T_M_ps || !d_cells) return proj_fail(PP_E_INVALID, "NULL argument");
    if (nM < 1 || nM > 8 || N_max < 1 || N_max > 65536) return proj_fail(PP_E_INVALID, "nM in [1,8], N_max in [1,65536]");
    if (sc->mini_batch == 0 || sc->dataset_items == 0 || sc->t1_ps == 0 || sc->ar_mode > 1)
        return proj_fail(PP_E_INVALID, "invalid scenario");
    if (sc->n_knots == 0 || sc->n_knots > kMaxKnots || !sc->knot_G || !sc->knot_uepochs)
        return proj_fail(PP_E_INVALID, "1..64 knots required");
    ProjParams P;
    memset(&P, 0, sizeof P);
    for (uint32_t i = 0; i < sc->n_knots; i++) {
        if (sc->knot_uepochs[i] == 0) return proj_fail(PP_E_INVALID, "knot epochs must be > 0");
        if (i > 0 && sc->knot_G[i] <= sc->knot_G[i - 1]) return proj_fail(PP_E_INVALID, "knot G must increase");
        if (i > 0) {
            uint64_t em = std::max(sc->knot_uepochs[i], sc->knot_uepochs[i - 1]);
            if (bitlen_h(em) + bitlen_h(sc->knot_G[i] - sc->knot_G[i - 1]) + 1 > 127)
                return proj_fail(PP_E_RANGE, "knot interpolation overflows 127 bits");
        }
        P.kG[i] = sc->knot_G[i];
        P.kE[i] = sc->knot_uepochs[i];
    }
    for (int m = 0; m < nM; m++) {
        if (Ms[m] == 0 || T_M_ps[m] == 0) return proj_fail(PP_E_INVALID, "M and T_M must be > 0");
        P.Ms[m] = Ms[m];
        P.TM[m] = T_M_ps[m];
    }
    P.D = sc->dataset_items;
    P.grad = sc->grad_bytes;
    P.bw_in = sc->bw_intra_Bps;
    P.lat_in = sc->lat_intra_ps;
    P.bw_out = sc->bw_inter_Bps;
    P.lat_out = sc->lat_inter_ps;
    P.t1 = sc->t1_ps;
    P.B = sc->mini_batch;
    P.n_knots = sc->n_knots;
    P.node = sc->node_size ? sc->node_size : 8;
    P.mode = sc->ar_mode;
    P.nM = (uint32_t)nM;
    P.N_max = N_max;
    if (sc->n_accum > kMaxAccum || (sc->n_accum && !sc->accum))
        return proj_fail(PP_E_INVALID, "n_accum in [0,32] with a host array");
    P.nA = sc->n_accum ? sc->n_accum : 1;
    P.A[0] = 1;
    for (uint32_t j = 0; j < sc->n_accum; j++) {
        if (sc->accum[j] == 0) return proj_fail(PP_E_INVALID, "accumulation factors must be >= 1");
        P.A[j] = sc->accum[j];
    }
    P.sharded = sc->shard_bytes != nullptr;
    if (P.sharded)
        for (int m = 0; m < nM; m++)
            for (int d = 0; d < 8; d++) P.shard[m][d] = sc->shard_bytes[8 * m + d];
    cudaStream_t st = (cudaStream_t)stream;
    ScratchSlot s(st);
    cudaError_t e = s.take();
    if (e == cudaSuccess) e = cudaMemsetAsync(s.p, 0, sizeof(int), st);
    if (e != cudaSuccess) return proj_fail(PP_E_CUDA, cudaGetErrorString(e));
    int *d_err = static_cast<int *>(s.p);
    int rc;
    if ((rc = launch_project(P, d_cells, d_err, stream))) return proj_fail(PP_E_CUDA, cudaGetErrorString((cudaError_t)rc));
    note_launch();
    int err = 0;
    e = cudaMemcpyAsync(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    s.synced = e == cudaSuccess;
    if (e != cudaSuccess) return proj_fail(PP_E_CUDA, cudaGetErrorString(e));
    if (err) return proj_fail(PP_E_RANGE, "projection value overflows 127 bits");
    return PP_OK;
}

extern "C" int pp_crossover(const pp_cell *d_cells, int nM, const uint32_t *Ms, uint32_t N_max,
                            pp_crossover_result *out, uint32_t *d_best_m, void *stream) {
    using namespace pp;
    if (!d_cells || !Ms || !out) return proj_fail(PP_E_INVALID, "NULL argument");
    if (nM < 1 || nM > 8 || N_max < 1 || N_max > 65536) return proj_fail(PP_E_INVALID, "nM in [1,8], N_max in [1,65536]");
    CrossParams X;
    memset(&X, 0, sizeof X);
    int m1 = -1;
    for (int m = 0; m < nM; m++) {
        X.Ms[m] = Ms[m];
        if (Ms[m] == 1) m1 = m;
    }
    if (m1 < 0) return proj_fail(PP_E_INVALID, "Ms must contain 1 (the DP-only baseline)");
    X.nM = (uint32_t)nM;
    X.N_max = N_max;
    X.m1 = (uint32_t)m1;
    cudaStream_t st = (cudaStream_t)stream;
    ScratchSlot s(st);
    static_assert(sizeof(pp_crossover_result) <= 256, "scratch slot size");
    cudaError_t e = s.take();
    if (e != cudaSuccess) return proj_fail(PP_E_CUDA, cudaGetErrorString(e));
    pp_crossover_result *d_x = static_cast<pp_crossover_result *>(s.p);
    int rc;
    if ((rc = launch_crossover(X, d_cells, d_x, d_best_m, stream))) return proj_fail(PP_E_CUDA, cudaGetErrorString((cudaError_t)rc));
    note_launch();
    e = cudaMemcpyAsync(out, d_x, sizeof *out, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    s.synced = e == cudaSuccess;
    if (e != cudaSuccess) return proj_fail(PP_E_CUDA, cudaGetErrorString(e));
    return PP_OK;
}
