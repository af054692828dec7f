// capi.cpp — the extern "C" entry points of libpp.so (include/pp.h): argument
// validation, launch configuration, the per-round search driver with the
// NCCL exchange, and the projection/crossover launches.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

typedef unsigned __int128 u128;

namespace pp {

static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};
static bool g_timing = false;
static double g_timing_ms = 0.0;
static uint64_t g_timing_n = 0;

void set_error(const std::string &msg) { g_err = msg; }
void note_launch() { g_launches++; }

int load_dfg(const pp_dfg_desc *d, const pp_link_desc *link, const pp_hw_desc *hw, int cuda_device, pp_dfg **out,
             pp_dfg_info *plan = nullptr, int32_t *plan_tier = nullptr);

#define PP_DECL_M(m)                                                                   \
    KernelInfo kernel_for_m##m(int gen, bool mem, bool wa, bool f64, int np, bool hw); \
    UpdateFn update_for_m##m(int gen);                                                 \
    XKernelInfo exact_for_m##m(int gen);                                              \
    KernelInfo big_for_m##m(int gen, bool f64);                                      \
    KernelInfo rp_kernel_for_m##m(bool mem, int np);
PP_DECL_M(1) PP_DECL_M(2) PP_DECL_M(3) PP_DECL_M(4) PP_DECL_M(5) PP_DECL_M(6) PP_DECL_M(7) PP_DECL_M(8)

KernelInfo kernel_for(int M, int gen, bool mem, bool wa, bool f64, int np, bool hw) {
    switch (M) {
        case 1: return kernel_for_m1(gen, mem, wa, f64, np, hw);
        case 2: return kernel_for_m2(gen, mem, wa, f64, np, hw);
        case 3: return kernel_for_m3(gen, mem, wa, f64, np, hw);
        case 4: return kernel_for_m4(gen, mem, wa, f64, np, hw);
        case 5: return kernel_for_m5(gen, mem, wa, f64, np, hw);
        case 6: return kernel_for_m6(gen, mem, wa, f64, np, hw);
        case 7: return kernel_for_m7(gen, mem, wa, f64, np, hw);
        default: return kernel_for_m8(gen, mem, wa, f64, np, hw);
    }
}
KernelInfo big_kernel_for(int M, int gen, bool f64) {
    switch (M) {
        case 1: return big_for_m1(gen, f64);
        case 2: return big_for_m2(gen, f64);
        case 3: return big_for_m3(gen, f64);
        case 4: return big_for_m4(gen, f64);
        case 5: return big_for_m5(gen, f64);
        case 6: return big_for_m6(gen, f64);
        case 7: return big_for_m7(gen, f64);
        default: return big_for_m8(gen, f64);
    }
}
static KernelInfo rp_kernel_for(int M, bool mem, int np) {
    return M == 2 ? rp_kernel_for_m2(mem, np) : M == 4 ? rp_kernel_for_m4(mem, np) : rp_kernel_for_m8(mem, np);
}
UpdateFn update_for(int M, int gen) {
    switch (M) {
        case 1: return update_for_m1(gen);
        case 2: return update_for_m2(gen);
        case 3: return update_for_m3(gen);
        case 4: return update_for_m4(gen);
        case 5: return update_for_m5(gen);
        case 6: return update_for_m6(gen);
        case 7: return update_for_m7(gen);
        default: return update_for_m8(gen);
    }
}

XKernelInfo exact_kernel_for(int M, int gen) {
    switch (M) {
        case 1: return exact_for_m1(gen);
        case 2: return exact_for_m2(gen);
        case 3: return exact_for_m3(gen);
        case 4: return exact_for_m4(gen);
        case 5: return exact_for_m5(gen);
        case 6: return exact_for_m6(gen);
        case 7: return exact_for_m7(gen);
        default: return exact_for_m8(gen);
    }
}

int launch_eft(const pp_dfg *g, int M, uint8_t *d_out, int *d_status, void *stream);

struct ProjParams;
struct CrossParams;
int launch_pack_key(uint64_t *s, int rank, void *stream);
int launch_patch_base(uint8_t *image, uint8_t *base, const uint8_t *src, uint32_t K, uint32_t K8, uint32_t off_hgw,
                      void *stream);
int launch_contrib(uint64_t *s, void *stream);
int launch_unpack_best(const uint64_t *s, uint64_t *out, void *stream);

static int cuda_err(cudaError_t e, const char *what) {
    set_error(std::string("CUDA: ") + what + ": " + cudaGetErrorString(e));
    return PP_E_CUDA;
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        err = cudaSetDevice(dev);
        ok = err == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// ------------------------------------------------------------ launch setup
struct Launch {
    KernelInfo k;
    int threads = 0, grid = 0, smem = 0, np = 0;
    KParams p{};
};

// Chooses NP (placements per lane), the CTA size and the dynamic shared
// memory layout, and a grid of (resident CTAs per SM) × SMs.  The per-warp
// state grows with W·NP, so for DFGs with many live values a smaller NP keeps
// more warps resident: take the largest NP that keeps ≥ 12 warps per SM (3
// per scheduler), else the NP with the most resident placements.
struct Choice {
    KernelInfo k;
    int np = 0, threads = 0, smem = 0, ctas = 0;
    uint32_t region = 0, slots_off = 0;
};

static int choose(const pp_dfg *g, int M, int gen, bool write_all, int np, Choice &c, bool rp = false) {
    const bool mem = g->cap > 0;
    c.k = rp ? rp_kernel_for(M, mem, np) : kernel_for(M, gen, mem, write_all, g->f64, np, g->hw);
    c.np = write_all ? 2 : np;
    const uint32_t nslot = (uint32_t)g->W + 1;                  // live + zero
    c.region = (nslot + (M > 2 ? (uint32_t)M : 0u)) * kSlotUnit * c.np;
    c.slots_off = (g->image_bytes + 127) & ~127u;
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, c.k.func);
    if (e != cudaSuccess) return cuda_err(e, "cudaFuncGetAttributes");
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device);
    const size_t max_dyn = (size_t)std::min<int>(optin, kMaxSmemBytes) - fa.sharedSizeBytes - 1024;
    // CTA size: the most resident warps per SM (each CTA holds its own copy
    // of the image), ties to the larger CTA; up to the kernel's launch bound
    c.threads = 0;
    int best_warps = 0;
    const int max_threads = std::min(fa.maxThreadsPerBlock, 1024) / 32 * 32;
    for (int threads = max_threads; threads >= 32; threads -= 32) {
        const size_t smem = c.slots_off + (size_t)(threads / 32) * c.region;
        if (smem > max_dyn) continue;
        e = cudaFuncSetAttribute(c.k.func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_err(e, "cudaFuncSetAttribute");
        int ctas = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, c.k.func, threads, (int)smem);
        if (e != cudaSuccess) return cuda_err(e, "occupancy");
        const int warps = ctas * threads / 32;
        if (ctas >= 1 && warps > best_warps) {
            best_warps = warps;
            c.threads = threads;
            c.smem = (int)smem;
            c.ctas = ctas;
        }
    }
    if (!c.threads) return PP_E_TOO_LARGE;
    e = cudaFuncSetAttribute(c.k.func, cudaFuncAttributeMaxDynamicSharedMemorySize, c.smem);
    if (e != cudaSuccess) return cuda_err(e, "cudaFuncSetAttribute");
    return PP_OK;
}

static void fill(const pp_dfg *g, const Choice &best, uint64_t begin, uint64_t end, Launch &L) {
    L.k = best.k;
    const uint64_t n = end - begin;
    const uint64_t per_warp = 32ull * best.np;
    const uint64_t tiles = (n + per_warp - 1) / per_warp;
    const uint64_t wpb = best.threads / 32;
    uint64_t want = (tiles + wpb - 1) / wpb;
    uint64_t grid = std::min<uint64_t>((uint64_t)best.ctas * g->sm_count, want);
    grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, kMaxGrid));
    L.threads = best.threads;
    L.grid = (int)grid;
    L.smem = best.smem;
    L.np = best.np;
    KParams &p = L.p;
    p.g_image = g->d_image;
    p.begin = begin;
    p.end = end;
    p.cap = g->cap;
    p.image_bytes = g->image_bytes;
    p.K = (uint32_t)g->K;
    p.K8 = (uint32_t)g->K8;
    p.off_extra = g->off_extra;
    p.off_mem = g->off_mem;
    p.off_orig = g->off_orig;
    p.smem_slots_off = best.slots_off;
    p.region_bytes = best.region;
    p.free_off = ((uint32_t)g->W + 1) * kSlotUnit;
    p.zero_off = (uint32_t)g->W * kSlotUnit;
    p.one_hi = 0x3FF00000u;
    p.off_cls = g->off_cls;
    p.off_hgw = g->off_hgw;
    p.g_partials = g->d_partials;
    p.g_ticket = g->d_ticket;
    p.g_tile = reinterpret_cast<unsigned long long *>(g->d_ticket + 4);
    p.g_out = g->d_scalars + SC_LOCAL_MK;
}

// Placements per lane (NP).  A rule fitted to the measured configurations
// (profiles/r01_np_rule.txt): with M ≤ 2 the most placements
// in flight (warps × NP, ties to more warps); with M ≥ 3, whose free[] lives
// in shared memory, the largest NP that keeps 20 warps per SM resident, else
// the most resident warps.
// PP_AUTOTUNE=1 instead times every NP variant on a probe range on the first
// call for a (DFG, M, generator) and keeps the fastest.  The result never
// depends on the choice (every variant is bit-exact), only the speed.
// The per-candidate (write-all) kernels are built for NP = 2 only.
// The global-state tier (pp_dfg::big): search_big_kernel with
// 256-thread CTAs, big_np(M) placements per lane, and a warp region of
// (W + 1 + M) slots × 256 B × big_np(M) in the DFG's global scratch.  The kernel uses no
// shared memory beyond its argmin scratch, so the L1 carve-out is maximal.
// Resident warps: the occupancy limit, unless the live state of all warps
// would exceed PP_BIG_STATE_MB (default 4096) of scratch.
static int setup_big(const pp_dfg *g, int M, int gen, bool write_all, uint64_t begin, uint64_t end, Launch &L) {
    if (gen == GEN_SYM) {
        set_error("symmetry-reduced search needs the shared-memory tier");
        return PP_E_TOO_LARGE;
    }
    L.k = big_kernel_for(M, gen, g->f64);
    constexpr int kThreads = 256;
    const uint64_t region = ((uint64_t)g->W + 1 + (M > 2 ? (uint64_t)M : 0ull)) * kSlotUnit * big_np(M);
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, L.k.func, kThreads, 0);
    if (e != cudaSuccess) return cuda_err(e, "occupancy");
    e = cudaFuncSetAttribute(L.k.func, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    if (e != cudaSuccess) return cuda_err(e, "cudaFuncSetAttribute carveout");
    uint64_t budget = 4096ull << 20;
    if (const char *v = getenv("PP_BIG_STATE_MB")) budget = std::max<uint64_t>(1, strtoull(v, nullptr, 10)) << 20;
    const uint64_t fit = budget / (region * (kThreads / 32) * (uint64_t)g->sm_count);
    per_sm = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)std::max(per_sm, 1), fit));
    const uint64_t n = end - begin;
    const uint64_t tiles = (n + 32 * big_np(M) - 1) / (32 * big_np(M));
    uint64_t grid = std::min<uint64_t>((uint64_t)per_sm * g->sm_count, (tiles + kThreads / 32 - 1) / (kThreads / 32));
    grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, kMaxGrid));
    const size_t need = (size_t)grid * (kThreads / 32) * region;
    pp_dfg *mg = const_cast<pp_dfg *>(g);
    if (need > mg->state_bytes) {   // grown on demand; cudaFree synchronises the device first
        if (mg->d_state) cudaFree(mg->d_state);
        mg->d_state = nullptr;
        mg->state_bytes = 0;
        if ((e = cudaMalloc(&mg->d_state, need)) != cudaSuccess) return cuda_err(e, "cudaMalloc state");
        mg->state_bytes = need;
    }
    L.threads = kThreads;
    L.grid = (int)grid;
    L.smem = 0;
    L.np = big_np(M);
    Choice c;
    c.k = L.k;
    c.np = big_np(M);
    c.threads = kThreads;
    c.ctas = per_sm;
    c.region = (uint32_t)region;
    c.slots_off = 0;
    fill(g, c, begin, end, L);
    L.grid = (int)grid;
    L.p.g_state = mg->d_state;
    L.p.g_makespan = nullptr;   // set by the write-all callers
    return PP_OK;
}

static int setup(const pp_dfg *g, int M, int gen, bool write_all, uint64_t begin, uint64_t end, Launch &L,
                 void *stream = nullptr, int force_np = 0) {
    if (g->big) return setup_big(g, M, gen, write_all, begin, end, L);
    int forced = force_np;   // PP_NP=1|2|4 pins NP (tests cover every variant)
    if (const char *v = getenv("PP_NP"); v && !forced) forced = atoi(v);
    std::vector<Choice> cands;
    for (int np : {4, 3, 2, 1}) {
        if (write_all && np != 2) continue;
        if (forced && np != forced) continue;
        if (np == 3 && !(gen == GEN_SYM && M == 3 && forced == 3)) continue;   // built for that case only
        Choice c;
        int rc = choose(g, M, gen, write_all, np, c);
        if (rc == PP_E_TOO_LARGE) continue;
        if (rc) return rc;
        cands.push_back(c);
    }
    if (cands.empty()) {
        set_error("per-lane schedule state does not fit in shared memory");
        return PP_E_TOO_LARGE;
    }
    size_t pick = 0;
    auto warps = [&](size_t i) { return (long)cands[i].ctas * cands[i].threads / 32; };
    if (M <= 2) {
        for (size_t i = 1; i < cands.size(); i++) {
            const long a = warps(i) * cands[i].np, b = warps(pick) * cands[pick].np;
            if (a > b || (a == b && warps(i) > warps(pick))) pick = i;
        }
    } else if (gen == GEN_PERTURB && (M == 4 || M == 8) && g->f64 && !g->hw) {
        // the device-word schedule (schedule_mpw): NP = 2 when it keeps ≥ 12
        // warps per SM — the fastest for every BASELINE DFG at M = 4 and 8
        // (profiles/r02_np_ab.txt) — else the most resident warps
        constexpr long kWarpMin = 12;
        bool found = false;
        for (size_t i = 0; i < cands.size() && !found; i++)
            if (cands[i].np == 2 && warps(i) >= kWarpMin) { pick = i; found = true; }
        if (!found)
            for (size_t i = 1; i < cands.size(); i++)
                if (warps(i) > warps(pick)) pick = i;
    } else {
        constexpr long kWarpTarget = 20;   // 5 per scheduler
        bool found = false;
        for (size_t i = 0; i < cands.size() && !found; i++)   // NP = 4, 2, 1 in order
            if (warps(i) >= kWarpTarget) { pick = i; found = true; }
        if (!found)
            for (size_t i = 1; i < cands.size(); i++)
                if (warps(i) > warps(pick)) pick = i;
    }
    const int key = (M << 8) | (gen << 4) | (write_all ? 1 : 0);
    auto it = g->tuned.find(key);
    const bool autotune = getenv("PP_AUTOTUNE") != nullptr;
    if (autotune && cands.size() > 1 && it != g->tuned.end()) {
        for (size_t i = 0; i < cands.size(); i++)
            if (cands[i].np == it->second) pick = i;
    } else if (autotune && cands.size() > 1) {
        // probe: the same candidate range for every variant, long enough to
        // fill the GPU a few times; each variant runs twice (the first run
        // absorbs module loading), the second is timed
        uint64_t probe = 0;
        for (auto &c : cands)
            probe = std::max<uint64_t>(probe, 4ull * c.ctas * g->sm_count * c.threads * c.np);
        probe = std::min<uint64_t>(probe, end - begin);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best_ms = 0;
        for (size_t i = 0; i < cands.size(); i++) {
            Launch T;
            fill(g, cands[i], begin, begin + probe, T);
            T.p.g_out = g->d_scalars + 40;          // scratch slots: no result is touched
            float ms = 0;
            for (int rep = 0; rep < 2; rep++) {
                cudaEventRecord(e0, (cudaStream_t)stream);
                int e = T.k.launch(T.p, T.grid, T.threads, T.smem, stream);
                g_launches++;
                cudaEventRecord(e1, (cudaStream_t)stream);
                if (e) { cudaEventDestroy(e0); cudaEventDestroy(e1); return cuda_err((cudaError_t)e, "probe"); }
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            if (i == 0 || ms < best_ms) { best_ms = ms; pick = i; }
            if (getenv("PP_VERBOSE"))
                fprintf(stderr, "pp: probe M=%d gen=%d np=%d threads=%d warps/SM=%d: %.3f ms\n", M, gen,
                        cands[i].np, cands[i].threads, cands[i].ctas * cands[i].threads / 32, ms);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        g->tuned[key] = cands[pick].np;
    }
    Choice best = cands[pick];
    // the PERTURB schedules with the next step's record prefetched (RP) when
    // few warps are resident (< 20 per SM, e.g. GNMT's 22 live values): GNMT
    // M = 4 +2.6%, while 24-warp configurations lose 0.3–1.4% to its extra
    // registers (profiles/r02_ab_rec_prefetch.txt).  PP_RP=0/1 overrides.
    if (gen == GEN_PERTURB && (M == 2 || M == 4 || M == 8) && g->f64 && !g->hw && !write_all) {
        const char *rv = getenv("PP_RP");
        const bool want = rv ? atoi(rv) != 0 : best.ctas * best.threads / 32 < 20;
        Choice c2;
        if (want && choose(g, M, gen, write_all, best.np, c2, true) == PP_OK) best = c2;
    }
    if (getenv("PP_VERBOSE")) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, best.k.func);
        fprintf(stderr, "pp: M=%d gen=%d np=%d threads=%d ctas/SM=%d warps/SM=%d smem=%d regs=%d W=%d\n", M, gen,
                best.np, best.threads, best.ctas, best.ctas * best.threads / 32, best.smem, fa.numRegs, g->W);
    }
    fill(g, best, begin, end, L);
    return PP_OK;
}

static int run(Launch &L, void *stream) {
    int e = L.k.launch(L.p, L.grid, L.threads, L.smem, stream);
    g_launches++;
    if (e != 0) return cuda_err((cudaError_t)e, "kernel launch");
    return PP_OK;
}

static int check_gen_args(const pp_dfg *g, int M, int gen, uint32_t tau, uint64_t end) {
    if (!g) { set_error("dfg is NULL"); return PP_E_INVALID; }
    if (M < 1 || M > 8) { set_error("M must be in [1,8]"); return PP_E_INVALID; }
    if (g->hw && M > g->nd) { set_error("M exceeds the hardware graph's devices"); return PP_E_INVALID; }
    if (gen < 0 || gen > 2) { set_error("unknown generator"); return PP_E_INVALID; }
    if (tau > 256) { set_error("flip_thresh must be in [0,256]"); return PP_E_INVALID; }
    if (gen == GEN_GRAY) {
        unsigned __int128 space = 1;
        for (int j = 0; j < g->K && space <= ((unsigned __int128)1 << 63); j++) space *= (unsigned)M;
        if (space > ((unsigned __int128)1 << 63)) { set_error("GRAY space M^K exceeds 2^63"); return PP_E_TOO_LARGE; }
        if ((unsigned __int128)end > space) { set_error("GRAY range exceeds M^K"); return PP_E_INVALID; }
    }
    return PP_OK;
}

// ------------------------------ symmetry-reduced exhaustive GRAY (f1)
// With the uniform link model the makespan and the memory feasibility of a
// placement are invariant under relabelling the devices, so an exhaustive
// GRAY search (the whole range [0, M^K)) evaluates one placement per class,
// the restricted-growth strings, and reports for each class that reaches the
// minimum its smallest Gray index (search_kernel.cuh RgsGen, gray_min_index;
// DESIGN.md §12b).  The (makespan, Gray index) argmin is the full search's.
// PP_NO_SYM=1 turns it off (A/B and tests).
static bool use_sym(const pp_dfg *g, int M, int gen, uint64_t begin, uint64_t end) {
    if (gen != GEN_GRAY || g->hw || g->big || M < 2 || g->K < 2 || begin != 0 || getenv("PP_NO_SYM")) return false;
    unsigned __int128 space = 1;
    for (int j = 0; j < g->K; j++) space *= (unsigned)M;   // ≤ 2^63 (check_gen_args)
    return (unsigned __int128)end == space;
}

// M = 2: the classes are pairs {d, d̄} (all K digits complemented), and with
// the reflected binary Gray code d = i ⊕ (i >> 1) the complement of d is the
// placement of i ⊕ c, c = the inverse Gray code of all ones (bits K−1, K−3,
// …).  c has bit K−1 set, so each class has exactly one index below 2^(K−1),
// and it is the class's smaller one: the plain GRAY search over the lower
// half [0, 2^(K−1)) returns the full search's (makespan, index) argmin at
// half the work and without the RGS unranking.

// Completion counts T_M[rem][m] = m·T_M[rem−1][m] + [m < M]·T_M[rem−1][m+1],
// T_M[0][m] = 1, for every M, uploaded once per DFG.  Returns the number of
// classes of M (= T_M[K−1][1]).
static int rgs_table(const pp_dfg *g, int M, uint64_t *classes) {
    const int rows = std::min(g->K, kRgsRows);
    if (!g->d_rgs) {
        std::vector<uint64_t> t((size_t)8 * kRgsRows * kRgsStride, 0);
        for (int mm = 1; mm <= 8; mm++) {
            uint64_t *T = t.data() + (size_t)(mm - 1) * kRgsRows * kRgsStride;
            for (int m = 1; m <= mm; m++) T[m] = 1;
            for (int r = 1; r < rows; r++)
                for (int m = 1; m <= mm; m++) {
                    unsigned __int128 v = (unsigned __int128)m * T[(r - 1) * kRgsStride + m];
                    if (m < mm) v += T[(r - 1) * kRgsStride + m + 1];
                    T[r * kRgsStride + m] = v >= ((unsigned __int128)1 << 63) ? (1ull << 63) : (uint64_t)v;
                }
        }
        uint64_t *d = nullptr;
        cudaError_t e = cudaMalloc(&d, t.size() * 8);
        if (e == cudaSuccess) e = cudaMemcpy(d, t.data(), t.size() * 8, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            if (d) cudaFree(d);
            return cuda_err(e, "RGS table");
        }
        g->d_rgs = d;
    }
    // T_M[K−1][1], recomputed on the host (exact: ≤ M^(K−1) < 2^63)
    std::vector<unsigned __int128> prev(M + 2, 1), cur(M + 2, 0);
    for (int r = 1; r < g->K; r++) {
        for (int m = 1; m <= M; m++) cur[m] = m * prev[m] + (m < M ? prev[m + 1] : 0);
        prev = cur;
    }
    *classes = (uint64_t)prev[1];
    return PP_OK;
}
static const uint64_t *rgs_of(const pp_dfg *g, int M) {
    return g->d_rgs + (size_t)(M - 1) * kRgsRows * kRgsStride;
}

// The in-order search kernel enumerates tasks: an RGS prefix of π positions
// 0..K−2 and a block of NP values of position K−1 (search_kernel.cuh).  NP is
// fixed first (PP_NP, else M for M ≤ 3 and 4 otherwise: the M values of the
// last position fill a lane), then tasks = (classes of K−1 positions)·⌈M/NP⌉.
static int sym_plan(const pp_dfg *g, int M, int *np, uint64_t *tasks) {
    int n = M <= 3 ? M : 4;
    if (const char *v = getenv("PP_NP")) {
        const int e = atoi(v);
        if (e == 1 || e == 2 || e == 4) n = e;
    }
    uint64_t classes = 0;
    int rc = rgs_table(g, M, &classes);
    if (rc) return rc;
    std::vector<unsigned __int128> prev(M + 2, 1), cur(M + 2, 0);
    for (int r = 1; r < g->K - 1; r++) {   // classes of the K−1 prefix positions
        for (int m = 1; m <= M; m++) cur[m] = m * prev[m] + (m < M ? prev[m + 1] : 0);
        prev = cur;
    }
    *np = n;
    *tasks = (uint64_t)prev[1] * (uint64_t)((M + n - 1) / n);
    return PP_OK;
}

// ------------------------------------------------------------------ NCCL
struct Nccl {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};

static Nccl *nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        n.CommInitRank = (decltype(n.CommInitRank))dlsym(h, "ncclCommInitRank");
        n.AllReduce = (decltype(n.AllReduce))dlsym(h, "ncclAllReduce");
        n.CommDestroy = (decltype(n.CommDestroy))dlsym(h, "ncclCommDestroy");
        n.GetErrorString = (decltype(n.GetErrorString))dlsym(h, "ncclGetErrorString");
        n.CommGetAsyncError = (decltype(n.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
        n.CommAbort = (decltype(n.CommAbort))dlsym(h, "ncclCommAbort");
        if (n.GetUniqueId && n.CommInitRank && n.AllReduce && n.CommDestroy && n.GetErrorString &&
            n.CommGetAsyncError && n.CommAbort)
            n.h = h;
    });
    return n.h ? &n : nullptr;
}

static int nccl_err(ncclResult_t r, const char *what) {
    Nccl *n = nccl();
    set_error(std::string("NCCL: ") + what + ": " + (n ? n->GetErrorString(r) : "unavailable"));
    return PP_E_NCCL;
}

}  // namespace pp

struct pp_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, device = 0;
    uint64_t timeout_ms = 0;     // 0: PP_NCCL_TIMEOUT_S or 600 s
    bool aborted = false;
};

namespace pp {

// The round exchange (protocol.h) on device scalars: the pack / contrib
// kernels and NCCL min all-reduces, all stream-ordered on st.
struct NcclExec {
    Nccl *nc;
    pp_comm *comm;
    uint64_t *s;
    cudaStream_t st;
    int pack() {
        int rc = launch_pack_key(s, comm->rank, st);
        g_launches++;
        return rc ? cuda_err((cudaError_t)rc, "pack") : PP_OK;
    }
    int contrib() {
        int rc = launch_contrib(s, st);
        g_launches++;
        return rc ? cuda_err((cudaError_t)rc, "contrib") : PP_OK;
    }
    int allreduce_min(int src, int dst) {
        ncclResult_t nr = nc->AllReduce(s + src, s + dst, 1, ncclUint64, ncclMin, comm->comm, st);
        return nr == ncclSuccess ? PP_OK : nccl_err(nr, "allreduce");
    }
};

// The same exchange on host scalars with a caller-supplied collective.
struct HostExec {
    uint64_t s[SC_COUNT];
    int rank;
    pp_allreduce_min_u64 fn;
    void *ctx;
    int pack() {
        s[SC_KEY_LOCAL] = proto::key(s[SC_LOCAL_MK], s[SC_LOCAL_IDX], rank);
        return PP_OK;
    }
    int contrib() {
        s[SC_IDX_LOCAL] = proto::contrib(s[SC_KEY_GLOBAL], s[SC_KEY_LOCAL], s[SC_LOCAL_IDX]);
        return PP_OK;
    }
    int allreduce_min(int src, int dst) {
        if (fn(ctx, s[src], &s[dst]) != 0) { set_error("allreduce callback failed"); return PP_E_NCCL; }
        return PP_OK;
    }
};

static uint64_t comm_timeout_ms(const pp_comm *c) {
    if (c && c->timeout_ms) return c->timeout_ms;
    if (const char *v = getenv("PP_NCCL_TIMEOUT_S")) {
        const long long t = atoll(v);
        if (t > 0) return (uint64_t)t * 1000;
    }
    return 600ull * 1000;
}

// Waits for st.  With a communicator, polls ncclCommGetAsyncError and the
// timeout while the stream is busy: a failed or dead peer aborts the comm
// (which also unblocks the stream) instead of hanging the caller.
static int wait_stream(cudaStream_t st, pp_comm *comm, Nccl *nc) {
    if (!comm) {
        cudaError_t e = cudaStreamSynchronize(st);
        return e == cudaSuccess ? PP_OK : cuda_err(e, "stream synchronize");
    }
    const uint64_t limit = comm_timeout_ms(comm);
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t spin = 0;; spin++) {
        cudaError_t q = cudaStreamQuery(st);
        if (q == cudaSuccess) return PP_OK;
        if (q != cudaErrorNotReady) return cuda_err(q, "stream query");
        ncclResult_t ae = ncclSuccess;
        nc->CommGetAsyncError(comm->comm, &ae);
        const uint64_t ms = (uint64_t)std::chrono::duration_cast<std::chrono::milliseconds>(
                                std::chrono::steady_clock::now() - t0).count();
        if ((ae != ncclSuccess && ae != ncclInProgress) || ms > limit) {
            nc->CommAbort(comm->comm);
            comm->comm = nullptr;
            comm->aborted = true;
            if (ae != ncclSuccess && ae != ncclInProgress) return nccl_err(ae, "asynchronous error (comm aborted)");
            set_error("NCCL: timeout after " + std::to_string(limit) + " ms (comm aborted)");
            return PP_E_NCCL;
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

}  // namespace pp

using namespace pp;

extern "C" {

const char *pp_last_error(void) { return g_err.c_str(); }
uint64_t pp_kernel_launch_count(void) { return g_launches.load(); }

void pp_set_kernel_timing(int enable) {
    g_timing = enable != 0;
    g_timing_ms = 0.0;
    g_timing_n = 0;
}

void pp_get_kernel_timing(double *total_ms, uint64_t *n) {
    if (total_ms) *total_ms = g_timing_ms;
    if (n) *n = g_timing_n;
}

int pp_plan_dfg(const pp_dfg_desc *desc, const pp_link_desc *link, pp_dfg_info *info, int32_t *tier) {
    if (!info) { set_error("info is NULL"); return PP_E_INVALID; }
    return load_dfg(desc, link, nullptr, 0, nullptr, info, tier);
}

int pp_load_dfg(const pp_dfg_desc *desc, const pp_link_desc *link, int cuda_device, pp_dfg **out) {
    g_err.clear();
    if (!link) { set_error("link is NULL"); return PP_E_INVALID; }
    return load_dfg(desc, link, nullptr, cuda_device, out);
}

int pp_load_dfg_hw(const pp_dfg_desc *desc, const pp_hw_desc *hw, int cuda_device, pp_dfg **out) {
    g_err.clear();
    if (!hw) { set_error("hw is NULL"); return PP_E_INVALID; }
    return load_dfg(desc, nullptr, hw, cuda_device, out);
}

int pp_dfg_get_info(const pp_dfg *g, pp_dfg_info *out) {
    if (!g || !out) { set_error("NULL argument"); return PP_E_INVALID; }
    out->num_ops = g->K;
    out->num_edges = g->E;
    out->num_slots = g->W;
    out->image_bytes = (int32_t)g->image_bytes;
    out->t1_ps = g->t1;
    out->grad_bytes = g->grad_bytes;
    return PP_OK;
}

int pp_dfg_get_tier(const pp_dfg *g) {
    if (!g) { set_error("NULL argument"); return PP_E_INVALID; }
    return g->big ? PP_TIER_GLOBAL : PP_TIER_SHARED;
}

int pp_dfg_get_pi(const pp_dfg *g, int32_t *pi_out) {
    if (!g || !pi_out) { set_error("NULL argument"); return PP_E_INVALID; }
    memcpy(pi_out, g->pi.data(), sizeof(int32_t) * g->K);
    return PP_OK;
}

int pp_eval_placements(const pp_dfg *g, int M, const uint8_t *d_placements, uint64_t count,
                       uint64_t *d_makespan, void *stream) {
    if (!g || M < 1 || M > 8 || (g->hw && M > g->nd) || (count && (!d_placements || !d_makespan))) {
        set_error("invalid arguments");
        return PP_E_INVALID;
    }
    if (count == 0) return PP_OK;
    DeviceGuard dg(g->device);
    if (!dg.ok) return cuda_err(dg.err, "cudaSetDevice");
    Launch L;
    int rc = setup(g, M, GEN_EXPLICIT, true, 0, count, L);
    if (rc) return rc;
    L.p.g_place = d_placements;
    L.p.g_makespan = d_makespan;
    return run(L, stream);
}

int pp_eval_generated(const pp_dfg *g, int M, int gen, uint64_t seed_r, uint32_t tau, const uint8_t *d_base_pi,
                      uint64_t begin, uint64_t count, uint64_t *d_makespan, void *stream) {
    int rc = check_gen_args(g, M, gen, tau, begin + count);
    if (rc) return rc;
    if (count == 0) return PP_OK;
    if (!d_makespan || (gen == GEN_PERTURB && !d_base_pi)) { set_error("NULL device buffer"); return PP_E_INVALID; }
    DeviceGuard dg(g->device);
    if (!dg.ok) return cuda_err(dg.err, "cudaSetDevice");
    if (gen == GEN_PERTURB) {
        if ((rc = launch_patch_base(g->d_image, g->d_base, d_base_pi, (uint32_t)g->K, (uint32_t)g->K8, g->off_hgw, stream)))
            return cuda_err((cudaError_t)rc, "base patch");
        g_launches++;
    }
    Launch L;
    rc = setup(g, M, gen, true, begin, begin + count, L);
    if (rc) return rc;
    L.p.seed = seed_r;
    L.p.tau = tau;
    L.p.g_makespan = d_makespan;
    return run(L, stream);
}

int pp_search_range(const pp_dfg *g, int M, int gen, uint64_t seed_r, uint32_t tau, const uint8_t *d_base_pi,
                    uint64_t begin, uint64_t end, uint64_t *d_best, void *stream) {
    int rc = check_gen_args(g, M, gen, tau, end);
    if (rc) return rc;
    if (end <= begin || !d_best || (gen == GEN_PERTURB && !d_base_pi)) {
        set_error("invalid range or NULL buffer");
        return PP_E_INVALID;
    }
    DeviceGuard dg(g->device);
    if (!dg.ok) return cuda_err(dg.err, "cudaSetDevice");
    if (gen == GEN_PERTURB) {
        if ((rc = launch_patch_base(g->d_image, g->d_base, d_base_pi, (uint32_t)g->K, (uint32_t)g->K8, g->off_hgw, stream)))
            return cuda_err((cudaError_t)rc, "base patch");
        g_launches++;
    }
    Launch L;
    if (use_sym(g, M, gen, begin, end) && M == 2) {   // the lower half of the Gray space (half_gray_space)
        if ((rc = setup(g, M, GEN_GRAY, false, 0, end / 2, L, stream))) return rc;
    } else if (use_sym(g, M, gen, begin, end)) {   // the whole GRAY space: one placement per class
        uint64_t tasks = 0;
        int np = 0;
        if ((rc = sym_plan(g, M, &np, &tasks))) return rc;
        if ((rc = setup(g, M, GEN_SYM, false, 0, tasks, L, stream, np))) return rc;
        L.p.g_rgs = rgs_of(g, M);
    } else if ((rc = setup(g, M, gen, false, begin, end, L, stream))) {
        return rc;
    }
    L.p.seed = seed_r;
    L.p.tau = tau;
    L.p.g_out = d_best;
    return run(L, stream);
}

// ------------------------------------------------ exact schedule (NEXT f1)
static constexpr uint64_t kDefaultNodeLimit = 1ull << 24;

static int run_exact(const pp_dfg *g, int M, int gen, uint64_t seed_r, uint32_t tau, const uint8_t *d_base_pi,
                     const uint8_t *d_place, uint64_t begin, uint64_t end, uint64_t node_limit,
                     uint64_t *d_makespan, uint8_t *d_exact, uint64_t *d_best, void *stream) {
    if (!g->x_bytes) {
        set_error("exact schedule needs 2K <= 64 nodes (K <= 32) and an image that fits");
        return PP_E_TOO_LARGE;
    }
    DeviceGuard dg(g->device);
    if (!dg.ok) return cuda_err(dg.err, "cudaSetDevice");
    const XKernelInfo k = exact_kernel_for(M, gen);
    const int threads = 256;
    const int ws_off = (int)((g->x_bytes + 15) & ~15u);
    const int smem = ws_off + (threads / 32) * (int)sizeof(XWarp);
    cudaError_t ce;
    if ((ce = cudaFuncSetAttribute(k.func, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess)
        return cuda_err(ce, "exact kernel attribute");
    int per_sm = 0;
    if ((ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k.func, threads, smem)) != cudaSuccess)
        return cuda_err(ce, "exact kernel occupancy");
    if (per_sm < 1) { set_error("exact kernel does not fit on an SM"); return PP_E_TOO_LARGE; }
    const uint64_t warps_needed = end - begin;
    uint64_t grid = (uint64_t)per_sm * (uint64_t)g->sm_count;
    const uint64_t by_work = (warps_needed + threads / 32 - 1) / (threads / 32);
    if (by_work < grid) grid = by_work;
    if (grid > (uint64_t)kMaxGrid) grid = kMaxGrid;
    if (grid < 1) grid = 1;
    cudaStream_t st = (cudaStream_t)stream;
    if ((ce = cudaMemsetAsync(g->d_xwork, 0, 4 * sizeof(unsigned long long), st)) != cudaSuccess ||
        (ce = cudaMemsetAsync(g->d_xwork + 1, 0xFF, sizeof(unsigned long long), st)) != cudaSuccess)
        return cuda_err(ce, "exact work counters");
    if (d_best && gen != GEN_EXPLICIT && !getenv("PP_NO_SEED_INC")) {
        // Seed the incumbent with the in-order argmin of the same candidates:
        // every placement's exact makespan is ≤ its in-order one, so the exact
        // optimum is ≤ that value, and pruning only trees whose bound is
        // strictly above it keeps every optimal placement (ties included).
        // The in-order kernel writes {makespan, index} to work[1], work[2];
        // work[2] (the unresolved count) is cleared again afterwards.
        const int igen = gen == GEN_SYM ? GEN_GRAY : gen;
        uint64_t ib = begin, ie = end;
        int rc;
        if (gen == GEN_PERTURB) {
            if ((rc = launch_patch_base(g->d_image, g->d_base, d_base_pi, (uint32_t)g->K, (uint32_t)g->K8,
                                        g->off_hgw, stream)))
                return cuda_err((cudaError_t)rc, "base patch");
            g_launches++;
        }
        Launch L;
        if (gen == GEN_SYM) {   // the classes stand for the whole Gray space
            int np = 0;
            if ((rc = sym_plan(g, M, &np, &ie))) return rc;
            ib = 0;
            if ((rc = setup(g, M, GEN_SYM, false, ib, ie, L, stream, np))) return rc;
            L.p.g_rgs = rgs_of(g, M);
        } else if ((rc = setup(g, M, igen, false, ib, ie, L, stream))) {
            return rc;
        }
        L.p.seed = seed_r;
        L.p.tau = tau;
        L.p.g_out = reinterpret_cast<uint64_t *>(g->d_xwork + 1);
        if ((rc = run(L, stream))) return rc;
        if ((ce = cudaMemsetAsync(g->d_xwork + 2, 0, sizeof(unsigned long long), st)) != cudaSuccess)
            return cuda_err(ce, "exact work counters");
    }
    XParams p{};
    p.g_ximage = g->d_ximage;
    p.g_place = d_place;
    p.g_base = d_base_pi;
    p.g_makespan = d_makespan;
    p.g_exact = d_exact;
    p.g_partials = g->d_partials;
    p.g_ticket = g->d_ticket;
    p.g_out = d_best;
    p.g_work = g->d_xwork;
    p.begin = begin;
    p.end = end;
    p.seed = seed_r;
    p.cap = g->cap;
    p.node_limit = node_limit ? node_limit : kDefaultNodeLimit;
    p.x_bytes = g->x_bytes;
    p.N = g->xN;
    p.K = (uint32_t)g->K;
    p.xcls = g->xcls;
    p.tau = tau;
    p.off_pred = g->x_off_pred;
    p.off_rows = g->x_off_rows;
    p.off_cls = g->x_off_cls;
    p.off_mem = g->x_off_mem;
    p.off_orig = g->x_off_orig;
    p.ws_off = (uint32_t)ws_off;
    p.search = d_best ? 1 : 0;
    p.g_rgs = gen == GEN_SYM ? rgs_of(g, M) : nullptr;
    int rc = k.launch(p, (int)grid, threads, smem, stream);
    g_launches++;
    if (rc) return cuda_err((cudaError_t)rc, "exact kernel launch");
    return PP_OK;
}

int pp_eval_exact(const pp_dfg *g, int M, const uint8_t *d_placements, uint64_t count, uint64_t node_limit,
                  uint64_t *d_makespan, uint8_t *d_exact, void *stream) {
    if (!g || M < 1 || M > 8 || (g->hw && M > g->nd) || (count && (!d_placements || !d_makespan))) {
        set_error("invalid arguments");
        return PP_E_INVALID;
    }
    if (count == 0) return PP_OK;
    return run_exact(g, M, GEN_EXPLICIT, 0, 0, nullptr, d_placements, 0, count, node_limit, d_makespan, d_exact,
                     nullptr, stream);
}

int pp_eval_exact_generated(const pp_dfg *g, int M, int gen, uint64_t seed_r, uint32_t tau,
                            const uint8_t *d_base_pi, uint64_t begin, uint64_t count, uint64_t node_limit,
                            uint64_t *d_makespan, uint8_t *d_exact, void *stream) {
    int rc = check_gen_args(g, M, gen, tau, begin + count);
    if (rc) return rc;
    if (count == 0) return PP_OK;
    if (!d_makespan || (gen == GEN_PERTURB && !d_base_pi)) { set_error("NULL device buffer"); return PP_E_INVALID; }
    return run_exact(g, M, gen, seed_r, tau, d_base_pi, nullptr, begin, begin + count, node_limit, d_makespan,
                     d_exact, nullptr, stream);
}

int pp_search_exact(const pp_dfg *g, int M, int gen, uint64_t seed_r, uint32_t tau, const uint8_t *d_base_pi,
                    uint64_t begin, uint64_t end, uint64_t node_limit, uint64_t *d_best, void *stream) {
    int rc = check_gen_args(g, M, gen, tau, end);
    if (rc) return rc;
    if (end <= begin || !d_best || (gen == GEN_PERTURB && !d_base_pi)) {
        set_error("invalid range or NULL buffer");
        return PP_E_INVALID;
    }
    if (use_sym(g, M, gen, begin, end) && M == 2)   // the lower half of the Gray space (half_gray_space)
        return run_exact(g, M, GEN_GRAY, seed_r, tau, d_base_pi, nullptr, 0, end / 2, node_limit, nullptr, nullptr,
                         d_best, stream);
    if (use_sym(g, M, gen, begin, end)) {   // the whole GRAY space: one placement per class
        uint64_t classes = 0;
        if ((rc = rgs_table(g, M, &classes))) return rc;
        return run_exact(g, M, GEN_SYM, seed_r, tau, d_base_pi, nullptr, 0, classes, node_limit, nullptr, nullptr,
                         d_best, stream);
    }
    return run_exact(g, M, gen, seed_r, tau, d_base_pi, nullptr, begin, end, node_limit, nullptr, nullptr, d_best,
                     stream);
}

// ------------------------------------------- pipeline-parallel MP (NEXT f3)
static uint64_t binom_sat(uint64_t n, uint64_t k) {   // C(n, k) saturating at 2^63
    if (k > n) return 0;
    unsigned __int128 c = 1;
    for (uint64_t i = 1; i <= k; i++) {
        c = c * (n - k + i) / i;
        if (c >= ((unsigned __int128)1 << 63)) return 1ull << 63;
    }
    return (uint64_t)c;
}

static int pipe_check(const pp_dfg *g, int M, const uint32_t *micro, int nm) {
    if (!g || M < 1 || M > 8 || !micro || nm < 1 || nm > 16) {
        set_error("M in [1,8], 1..16 micro-batch counts");
        return PP_E_INVALID;
    }
    if (g->hw) { set_error("pipeline evaluation uses the uniform link (not a hardware graph)"); return PP_E_INVALID; }
    if (M > g->K) { set_error("more stages than ops"); return PP_E_INVALID; }
    if (g->K > kMaxPipelineK) { set_error("pipeline evaluation supports K <= 1024"); return PP_E_TOO_LARGE; }
    for (int j = 0; j < nm; j++)
        if (micro[j] < 1 || micro[j] > 65536) { set_error("micro-batch counts in [1,65536]"); return PP_E_INVALID; }
    return PP_OK;
}

// Range of the pipeline arithmetic (u64 in the kernel): with m micro-batches
// and a per-op overhead o, every stage time is ≤ ⌈ΣΔ/m⌉ + K·o and every
// transfer ≤ ⌈D·10^12/(m·BW)⌉ + L, and the makespan is a longest path
// through ≤ 2·m·M stage slots and ≤ 2·m·M transfers, so
//   makespan ≤ T_1 + 2·m·M·(K·o + 1) + 2·M·(Σ_e c_e) + 2·m·M·(L + 1).
// That bound, the π-prefix sums of M(k) and the 2-D byte prefix sums must
// stay below 2^63, else PP_E_RANGE (the loader's 2^61 bound covers only the
// placement schedule).
static int pipe_range(const pp_dfg *g, int M, const uint32_t *micro, int nm, uint64_t overhead) {
    uint64_t mx = 0;
    for (int j = 0; j < nm; j++) mx = std::max<uint64_t>(mx, micro[j]);
    u128 comm = 0, bytes = 0, mem = 0;
    for (size_t e = 0; e < g->e_src.size(); e++) {
        bytes += (u128)g->e_bf[e] + g->e_bb[e];
        comm += ((u128)g->e_bf[e] * 1000000000000ull + g->link_bw - 1) / g->link_bw;
        comm += ((u128)g->e_bb[e] * 1000000000000ull + g->link_bw - 1) / g->link_bw;
    }
    for (int p = 0; p < g->K; p++) mem += g->mem[p];
    const u128 lim = (u128)1 << 63;
    if (overhead >= lim / ((u128)g->K + 1) || comm >= lim || bytes >= lim || mem >= lim) {
        set_error("pipeline arithmetic exceeds 2^63");
        return PP_E_RANGE;
    }
    const u128 bound = (u128)g->t1 + 2 * (u128)mx * M * ((u128)g->K * overhead + 1) + 2 * (u128)M * comm +
                       2 * (u128)mx * M * ((u128)g->link_lat + 1);
    if (bound >= lim) {
        set_error("pipeline makespan bound exceeds 2^63 ps");
        return PP_E_RANGE;
    }
    return PP_OK;
}

static int pipe_tables(pp_dfg *g) {
    if (g->d_pipe) return PP_OK;
    const uint64_t K1 = (uint64_t)g->K + 1;
    std::vector<uint64_t> h(3 * K1 + 3 * K1 * K1 + K1 * 8, 0);
    uint64_t *pf = h.data(), *pb = pf + K1, *pm = pb + K1, *qf = pm + K1, *qb = qf + K1 * K1, *qc = qb + K1 * K1,
             *bn = qc + K1 * K1;
    for (int p = 0; p < g->K; p++) {
        pf[p + 1] = pf[p] + g->fwd[p];
        pb[p + 1] = pb[p] + g->bwd[p];
        pm[p + 1] = pm[p] + g->mem[p];
    }
    for (size_t e = 0; e < g->e_src.size(); e++) {
        const uint64_t at = (uint64_t)(g->e_src[e] + 1) * K1 + (uint64_t)(g->e_dst[e] + 1);
        qf[at] += g->e_bf[e];
        qb[at] += g->e_bb[e];
        qc[at] += 1;
    }
    for (uint64_t i = 1; i < K1; i++)
        for (uint64_t j = 1; j < K1; j++) {
            const uint64_t a = i * K1 + j, l = i * K1 + j - 1, u = (i - 1) * K1 + j, ul = (i - 1) * K1 + j - 1;
            qf[a] += qf[l] + qf[u] - qf[ul];
            qb[a] += qb[l] + qb[u] - qb[ul];
            qc[a] += qc[l] + qc[u] - qc[ul];
        }
    for (uint64_t n = 0; n < K1; n++)
        for (uint64_t k = 0; k < 8; k++) bn[n * 8 + k] = binom_sat(n, k);
    cudaError_t ce;
    if ((ce = cudaMalloc(&g->d_pipe, h.size() * 8)) != cudaSuccess) return cuda_err(ce, "pipeline tables");
    if ((ce = cudaMemcpy(g->d_pipe, h.data(), h.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_err(ce, "pipeline tables");
    return PP_OK;
}

int pp_pipeline_space(const pp_dfg *g, int M, int nm, uint64_t *count) {
    if (!g || M < 1 || M > 8 || M > g->K || nm < 1 || nm > 16 || !count) {
        set_error("invalid arguments");
        return PP_E_INVALID;
    }
    const unsigned __int128 c = (unsigned __int128)binom_sat((uint64_t)g->K - 1, (uint64_t)M - 1) * (unsigned)nm;
    if (c >= ((unsigned __int128)1 << 63)) { set_error("pipeline space exceeds 2^63"); return PP_E_TOO_LARGE; }
    *count = (uint64_t)c;
    return PP_OK;
}

int pp_pipeline_range(const pp_dfg *gc, int M, const uint32_t *micro, int nm, uint64_t overhead_ps, uint64_t begin,
                      uint64_t end, uint64_t *d_best, uint64_t *d_makespan, void *stream) {
    int rc = pipe_check(gc, M, micro, nm);
    if (rc) return rc;
    if ((rc = pipe_range(gc, M, micro, nm, overhead_ps))) return rc;
    uint64_t space = 0;
    if ((rc = pp_pipeline_space(gc, M, nm, &space))) return rc;
    if (end <= begin || end > space || (!d_best && !d_makespan)) {
        set_error("invalid range or no output");
        return PP_E_INVALID;
    }
    pp_dfg *g = const_cast<pp_dfg *>(gc);   // the tables are a cache
    DeviceGuard dg(g->device);
    if (!dg.ok) return cuda_err(dg.err, "cudaSetDevice");
    if ((rc = pipe_tables(g))) return rc;
    const uint64_t K1 = (uint64_t)g->K + 1;
    PipeParams p{};
    p.g_pf = g->d_pipe;
    p.g_pb = p.g_pf + K1;
    p.g_pm = p.g_pb + K1;
    p.g_qf = p.g_pm + K1;
    p.g_qb = p.g_qf + K1 * K1;
    p.g_qc = p.g_qb + K1 * K1;
    p.g_binom = p.g_qc + K1 * K1;
    p.g_makespan = d_makespan;
    p.g_partials = g->d_partials;
    p.g_ticket = g->d_ticket;
    p.g_out = d_best;
    p.bw = g->link_bw;
    p.lat = g->link_lat;
    p.cap = g->cap;
    p.begin = begin;
    p.end = end;
    p.K = (uint32_t)g->K;
    p.nm = (uint32_t)nm;
    p.overhead = overhead_ps;
    for (int j = 0; j < nm; j++) p.micro[j] = micro[j];
    const int threads = pipeline_block_threads(M);
    const uint64_t ranks = (end + nm - 1) / nm - begin / nm;
    uint64_t grid = (uint64_t)g->sm_count * 8;
    const uint64_t want = (ranks + threads - 1) / threads;
    if (want < grid) grid = want;
    if (grid < 1) grid = 1;
    if (grid > (uint64_t)kMaxGrid) grid = kMaxGrid;
    p.block = (ranks + grid * threads - 1) / (grid * threads);
    if (p.block < 1) p.block = 1;
    rc = launch_pipeline(M, p, (int)grid, stream);
    g_launches++;
    if (rc) return cuda_err((cudaError_t)rc, "pipeline kernel launch");
    return PP_OK;
}

int pp_pipeline_search(const pp_dfg *g, int M, const uint32_t *micro, int nm, uint64_t overhead_ps, void *stream,
                       pp_pipeline_result *out) {
    if (!out) { set_error("out is NULL"); return PP_E_INVALID; }
    int rc = pipe_check(g, M, micro, nm);
    if (rc) return rc;
    uint64_t space = 0;
    if ((rc = pp_pipeline_space(g, M, nm, &space))) return rc;
    DeviceGuard dg(g->device);
    if (!dg.ok) return cuda_err(dg.err, "cudaSetDevice");
    uint64_t *d_best = g->d_scalars + 32;    // scratch slots 32, 33
    if ((rc = pp_pipeline_range(g, M, micro, nm, overhead_ps, 0, space, d_best, nullptr, stream))) return rc;
    uint64_t best[2];
    cudaError_t ce;
    if ((ce = cudaMemcpyAsync(best, d_best, sizeof best, cudaMemcpyDeviceToHost, (cudaStream_t)stream)) !=
            cudaSuccess ||
        (ce = cudaStreamSynchronize((cudaStream_t)stream)) != cudaSuccess)
        return cuda_err(ce, "pipeline result");
    memset(out, 0, sizeof *out);
    out->makespan_ps = best[0];
    out->index = best[1];
    out->candidates = space;
    out->n_stages = (uint32_t)M;
    out->micro_batches = micro[best[1] % (uint64_t)nm];
    uint64_t rank = best[1] / (uint64_t)nm;       // unrank the cut vector
    uint64_t x = 1;
    for (int i = 0; i < M - 1; i++) {
        for (;;) {
            const uint64_t c = binom_sat((uint64_t)g->K - 1 - x, (uint64_t)(M - 2 - i));
            if (rank < c) break;
            rank -= c;
            x++;
        }
        out->cuts[i] = (int32_t)x;
        x++;
    }
    if (best[0] == PP_INFEASIBLE_MAKESPAN) {
        set_error("every pipeline violates the device memory capacity");
        return PP_E_INFEASIBLE;
    }
    return PP_OK;
}

// ------------------------------------- placement-aware AR shards (NEXT f4)
int pp_shard_bytes(const pp_dfg *g, int M, const uint8_t *placement, uint64_t *out) {
    if (!g || M < 1 || M > 8 || !placement || !out) {
        set_error("invalid arguments");
        return PP_E_INVALID;
    }
    for (int d = 0; d < 8; d++) out[d] = 0;
    for (int k = 0; k < g->K; k++) {
        if (placement[k] >= M) { set_error("placement value >= M"); return PP_E_INVALID; }
        out[placement[k]] += g->param[k];
    }
    return PP_OK;
}

// ------------------------------------------------- EFT base seed (NEXT f4)
int pp_eft_place(const pp_dfg *g, int M, uint8_t *placement, void *stream) {
    if (!g || M < 1 || M > 8 || (g->hw && M > g->nd) || !placement) {
        set_error("invalid arguments");
        return PP_E_INVALID;
    }
    DeviceGuard dg(g->device);
    if (!dg.ok) return cuda_err(dg.err, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    // scratch: the placement in d_winner, the status in the ticket slot 2
    int *d_status = reinterpret_cast<int *>(g->d_ticket + 2);
    int rc = launch_eft(g, M, g->d_winner, d_status, stream);
    g_launches++;
    if (rc) return cuda_err((cudaError_t)rc, "EFT kernel launch");
    std::vector<uint8_t> pl(g->K);
    int status = 0;
    cudaError_t ce;
    if ((ce = cudaMemcpyAsync(pl.data(), g->d_winner, g->K, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (ce = cudaMemcpyAsync(&status, d_status, sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (ce = cudaStreamSynchronize(st)) != cudaSuccess)
        return cuda_err(ce, "EFT result");
    if (status) {
        set_error("no memory-feasible device for some op");
        return PP_E_INFEASIBLE;
    }
    for (int p = 0; p < g->K; p++) placement[g->pi[p]] = pl[p];
    return PP_OK;
}

void pp_rank_slice(uint64_t count, int rank, int world, uint64_t *begin, uint64_t *end) {
    unsigned __int128 c = count;
    *begin = (uint64_t)(c * (unsigned)rank / (unsigned)world);
    *end = (uint64_t)(c * (unsigned)(rank + 1) / (unsigned)world);
}

uint64_t pp_pack_key(uint64_t makespan, int rank) { return proto::key(makespan, 0, rank); }
uint64_t pp_key_makespan(uint64_t key) { return proto::key_makespan(key); }
int pp_key_rank(uint64_t key) { return proto::key_rank(key); }

int pp_search_best(const pp_dfg *g, int M, const pp_search_desc *desc, pp_comm *comm, void *stream,
                   pp_search_result *out) {
    g_err.clear();
    if (!desc || !out) { set_error("NULL argument"); return PP_E_INVALID; }
    int rc = check_gen_args(g, M, desc->gen, desc->flip_thresh, desc->count);
    if (rc) return rc;
    if (desc->count < 1 || desc->rounds < 1 || (desc->gen != GEN_PERTURB && desc->rounds != 1)) {
        set_error("count must be >= 1; rounds must be >= 1 and > 1 only for PERTURB");
        return PP_E_INVALID;
    }
    const int rank = comm ? comm->rank : 0, world = comm ? comm->world : 1;
    if (world < 1 || world > 8) { set_error("1 to 8 ranks"); return PP_E_INVALID; }
    if (comm && comm->aborted) { set_error("communicator was aborted"); return PP_E_NCCL; }
    Nccl *nc = comm ? nccl() : nullptr;
    if (comm && !nc) { set_error("NCCL not loadable"); return PP_E_NCCL; }
    DeviceGuard dg(g->device);
    if (!dg.ok) return cuda_err(dg.err, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    const int K = g->K;
    // base (π order)
    std::vector<uint8_t> base(g->base_bytes, 0);
    if (desc->base)
        for (int p = 0; p < K; p++) {
            base[p] = desc->base[g->pi[p]];
            if (base[p] >= M) { set_error("base device out of range"); return PP_E_INVALID; }
        }
    cudaError_t e = cudaMemcpyAsync(g->d_winner, base.data(), g->base_bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_err(e, "base upload");
    if ((rc = launch_patch_base(g->d_image, g->d_base, g->d_winner, (uint32_t)K, (uint32_t)g->K8, g->off_hgw, stream)))
        return cuda_err((cudaError_t)rc, "base patch");
    g_launches++;
    // an exhaustive GRAY search runs over the relabelling classes (f1); its
    // winner is reported by Gray index, so the update is GRAY's
    const bool half = use_sym(g, M, desc->gen, 0, desc->count) && M == 2;   // half_gray_space
    const bool sym = use_sym(g, M, desc->gen, 0, desc->count) && !half;
    uint64_t space = half ? desc->count / 2 : desc->count;
    int sym_np = 0;
    if (sym && (rc = sym_plan(g, M, &sym_np, &space))) return rc;
    uint64_t begin = 0, end = 0;
    pp_rank_slice(space, rank, world, &begin, &end);
    UpdateFn upd = update_for(M, desc->gen);
    Launch L;
    const bool empty = end <= begin;
    if (!empty) {
        rc = setup(g, M, sym ? GEN_SYM : desc->gen, false, begin, end, L, stream, sym_np);
        if (rc) return rc;
        L.p.tau = desc->flip_thresh;
        if (sym) L.p.g_rgs = rgs_of(g, M);
    }
    std::vector<cudaEvent_t> evs;
    struct EvGuard {
        std::vector<cudaEvent_t> &v;
        ~EvGuard() {
            for (cudaEvent_t x : v) cudaEventDestroy(x);
        }
    } evg{evs};
    for (uint32_t r = 0; r < desc->rounds; r++) {
        const uint64_t seed_r = desc->seed + r;
        if (!empty) {
            L.p.seed = seed_r;
            if (g_timing) {
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                evs.push_back(a);
                evs.push_back(b);
                cudaEventRecord(a, st);
            }
            if ((rc = run(L, stream))) return rc;
            if (g_timing) cudaEventRecord(evs.back(), st);
        } else {
            uint64_t none[2] = {PP_INFEASIBLE_MAKESPAN, PP_INFEASIBLE_MAKESPAN};
            e = cudaMemcpyAsync(g->d_scalars + SC_LOCAL_MK, none, sizeof none, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) return cuda_err(e, "empty slice");
            cudaStreamSynchronize(st);
        }
        if (comm) {
            // the round exchange (protocol.h): packed-key min all-reduce picks
            // the winning rank, a second min all-reduce delivers its index
            NcclExec ex{nc, comm, g->d_scalars, st};
            if ((rc = proto::exchange(ex))) return rc;
        }
        UParams u{g->d_image, g->d_base, g->d_winner, g->d_best_place, g->d_scalars, seed_r, (uint32_t)K,
                  (uint32_t)g->K8, desc->flip_thresh,
                  r, comm ? 1 : 0, g->off_hgw};
        if ((rc = upd(u, stream))) return cuda_err((cudaError_t)rc, "round update");
        g_launches++;
    }
    uint64_t best[3];
    std::vector<uint8_t> place(g->base_bytes);
    e = cudaMemcpyAsync(best, g->d_scalars + SC_BEST_MK, sizeof best, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(place.data(), g->d_best_place, g->base_bytes, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_err(e, "search result");
    if ((rc = wait_stream(st, comm, nc))) return rc;
    for (size_t i = 0; i + 1 < evs.size(); i += 2) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, evs[i], evs[i + 1]) == cudaSuccess) {
            g_timing_ms += ms;
            g_timing_n++;
        }
    }
    out->best_makespan_ps = best[0];
    out->best_index = best[1];
    out->best_round = best[2];
    out->t1_ps = g->t1;
    out->evaluated = desc->count * (uint64_t)desc->rounds;
    if (out->placement)
        for (int p = 0; p < K; p++) out->placement[g->pi[p]] = place[p];
    if (best[0] == PP_INFEASIBLE_MAKESPAN) {
        set_error("every candidate violates the device memory capacity");
        return PP_E_INFEASIBLE;
    }
    return PP_OK;
}

int pp_argmin_allreduce(const pp_dfg *g, pp_comm *comm, uint64_t *d_best, void *stream) {
    if (!g || !comm || !d_best) { set_error("invalid arguments"); return PP_E_INVALID; }
    if (comm->aborted) { set_error("communicator was aborted"); return PP_E_NCCL; }
    Nccl *nc = nccl();
    if (!nc) { set_error("NCCL not loadable"); return PP_E_NCCL; }
    DeviceGuard dg(g->device);
    if (!dg.ok) return cuda_err(dg.err, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(g->d_scalars + SC_LOCAL_MK, d_best, 2 * sizeof(uint64_t),
                                    cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_err(e, "argmin copy");
    NcclExec ex{nc, comm, g->d_scalars, st};
    int rc;
    if ((rc = proto::exchange(ex))) return rc;
    if ((rc = launch_unpack_best(g->d_scalars, d_best, stream))) return cuda_err((cudaError_t)rc, "unpack");
    g_launches++;
    return wait_stream(st, comm, nc);
}

int pp_comm_set_timeout(pp_comm *comm, uint64_t timeout_ms) {
    if (!comm) { set_error("NULL comm"); return PP_E_INVALID; }
    comm->timeout_ms = timeout_ms;
    return PP_OK;
}

uint64_t pp_round_key(uint64_t makespan, uint64_t index, int rank) { return proto::key(makespan, index, rank); }
uint64_t pp_round_contrib(uint64_t key_global, uint64_t key_local, uint64_t local_index) {
    return proto::contrib(key_global, key_local, local_index);
}
int pp_round_moves_base(uint64_t win_index) { return proto::moves_base(win_index) ? 1 : 0; }

int pp_round_exchange_host(uint64_t local_makespan, uint64_t local_index, int rank, pp_allreduce_min_u64 fn,
                           void *ctx, uint64_t win[2]) {
    if (!fn || !win || rank < 0 || rank > 7) { set_error("invalid arguments"); return PP_E_INVALID; }
    HostExec ex{};
    ex.s[SC_LOCAL_MK] = local_makespan;
    ex.s[SC_LOCAL_IDX] = local_index;
    ex.rank = rank;
    ex.fn = fn;
    ex.ctx = ctx;
    int rc = proto::exchange(ex);
    if (rc) return rc;
    win[0] = proto::key_makespan(ex.s[SC_KEY_GLOBAL]);
    win[1] = ex.s[SC_IDX_GLOBAL];
    return PP_OK;
}

int pp_comm_get_unique_id(uint8_t out_id[128]) {
    Nccl *n = nccl();
    if (!n) { set_error("NCCL not loadable"); return PP_E_NCCL; }
    ncclUniqueId id;
    ncclResult_t r = n->GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_err(r, "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out_id, &id, 128);
    return PP_OK;
}

int pp_comm_init(const uint8_t id_bytes[128], int rank, int world, int cuda_device, pp_comm **out) {
    if (!out || !id_bytes || world < 1 || world > 8 || rank < 0 || rank >= world) {
        set_error("invalid comm arguments (1..8 ranks)");
        return PP_E_INVALID;
    }
    Nccl *n = nccl();
    if (!n) { set_error("NCCL not loadable"); return PP_E_NCCL; }
    DeviceGuard dg(cuda_device);
    if (!dg.ok) return cuda_err(dg.err, "cudaSetDevice");
    ncclUniqueId id;
    memcpy(&id, id_bytes, 128);
    pp_comm *c = new pp_comm();
    ncclResult_t r = n->CommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) { delete c; return nccl_err(r, "ncclCommInitRank"); }
    c->rank = rank;
    c->world = world;
    c->device = cuda_device;
    *out = c;
    return PP_OK;
}

void pp_comm_destroy(pp_comm *c) {
    if (!c) return;
    Nccl *n = nccl();
    if (n && c->comm && !c->aborted) n->CommDestroy(c->comm);
    delete c;
}

}  // extern "C"
