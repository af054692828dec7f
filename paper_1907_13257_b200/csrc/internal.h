// internal.h — shared declarations of libpp.so (not part of the C ABI).
//
// The shared-memory image (built by loader.cpp, read by search_kernel.cuh):
//
//   [OpRec   × 2K8]  one 32-B record per scheduled op, in issue order: steps
//                    s = 0..K8−1 are the forward ops of π positions p = s, steps
//                    s = K8..2K8−1 the backward ops of p = 2K8−1−s (readings
//                    R1/R2).  K8 = K rounded up to a multiple of 8; positions
//                    p ≥ K are no-op pads (zero cost, zero input) that leave
//                    every device's free time unchanged.
//                    The op's FIRST input edge is inlined in the record (most
//                    ops of a training DFG have in-degree 1); an op without
//                    inputs gets a zero-cost edge from the always-zero slot, a
//                    sink's backward gets a zero-cost "self" edge from its own
//                    forward finish time (it waits for its own forward, R1).
//   [ExtraRec × NX]  the remaining input edges, consumed in step order.
//   [u64   × K8 ]    M(k) by π position (read only when a memory cap is set)
//   [u32   × K8 ]    descriptor index of π position p (explicit placements)
//   [u32   × K8/4]   PERTURB base of each half-group (π positions 4h..4h+3):
//                    byte c = base device of position 4h + c (pads: 0), read
//                    by the M = 4, 8 device-word schedule (search_kernel.cuh)
//   [u8    × 64 ]    hardware graph only: cost class of device pair (a, b)
//   [u64 × rows·C]   hardware graph only: per-input cost rows, one f64-encoded
//                    cost per class (class 0 = same device, unused); the
//                    records' cost fields then hold the row's byte offset
//
// Per-lane schedule state lives in a per-warp region of shared memory laid out
// [slot][placement k < NP][lane] × u64, so a slot's byte offset inside the
// region is slot·256·NP (the records hold slot·256) and every access of a
// warp touches 32 consecutive u64 (conflict-free).  Slots 0..W−1 hold
// live finish times (liveness-allocated), slot W is always zero.  An input
// produced by the immediately preceding step is forwarded in a register
// (kFromPrev) and a value that no later step reads from a slot is not stored.
//
// Times in the kernel are TAGGED with the producer's device, so one slot read
// yields both a finish time and its device:
//   u64 arithmetic: value = 8·t + device (t < 2^61);
//   f64 arithmetic (all times < 2^49): value = the double t with the device in
//   its 3 low mantissa bits, i.e. t + device·ulp(t) — integers below 2^49 have
//   those bits clear, adds of integers stay exact, and the tag never reaches
//   the integer part.
// A max over tagged values has the max time in its integer part (ties differ
// only in the tag, which is cleared before use).
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../../include/pp.h"
#include "protocol.h"

namespace pp {

// Slot offsets in the image are in units of kSlotUnit = 256 bytes (one u64
// per lane of a warp); a kernel evaluating NP placements per lane (NP ∈ {1,
// 2, 4}, chosen per launch from W and shared memory) scales them by NP.
constexpr uint32_t kSlotUnit = 256u;

constexpr uint32_t kFromPrev = 0xFFFFFFFFu;     // OpRec.src_off: previous step's output (register)
constexpr uint32_t kNoStore = 0xFFFFFFFFu;      // OpRec.out_off: output never read from a slot

// cost8 / c8 / ExtraRec.c8 hold the ENCODED cost: 8·ps for the tagged-u64
// arithmetic, the bits of (double)ps for the tagged-f64 arithmetic.
struct OpRec {
    uint64_t cost8;       // encoded Δf(p) or Δb(p)
    uint64_t c8;          // encoded c of the first input edge (0 for the zero / self edge)
    uint32_t src_off;     // region byte offset of the first input's slot, or kFromPrev
    uint32_t out_off;     // region byte offset of the output slot, or kNoStore
    uint32_t ctrl;        // 0: fast chain step (first input = previous step, no extras);
                          // else 0x10000 | n_extra (further inputs, ExtraRec in order)
    uint32_t base;        // PERTURB base (patched every round): bits 0..2 the base device
                          // of this op; bits 7, 15, 23, 31 bit 0 of the base devices of
                          // the 4 ops of its half-group (π positions 4h..4h+3), read by
                          // the M = 2 cut-word schedule (search_kernel.cuh)
};
static_assert(sizeof(OpRec) == 32, "OpRec is 32 B");

struct ExtraRec {
    uint64_t c8;          // 8·c(e) (c = ⌈D·10^12/BW⌉ + L)
    uint32_t src_off;     // region byte offset of the producer's slot
    uint32_t pad;
};
static_assert(sizeof(ExtraRec) == 16, "ExtraRec is 16 B");

// The packed half-group word of π position p: bit 8c+7 = bit 0 of the base
// device of position 4⌊p/4⌋ + c (positions ≥ K, the no-op pads, count as 0).
#ifdef __CUDACC__
__host__ __device__ __forceinline__
#else
inline
#endif
uint32_t half_group_word(const uint8_t *base, uint32_t p, uint32_t K) {
    uint32_t w = 0;
    for (uint32_t c = 0; c < 4; c++) {
        const uint32_t q = (p & ~3u) + c;
        if (q < K) w |= (uint32_t)(base[q] & 1u) << (8 * c + 7);
    }
    return w;
}

// The half-group base word of half-group h: byte c = base device of π
// position 4h + c (positions ≥ K count as device 0).
#ifdef __CUDACC__
__host__ __device__ __forceinline__
#else
inline
#endif
uint32_t half_group_bytes(const uint8_t *base, uint32_t h, uint32_t K) {
    uint32_t w = 0;
    for (uint32_t c = 0; c < 4; c++) {
        const uint32_t q = 4 * h + c;
        if (q < K) w |= (uint32_t)(base[q] & 7u) << (8 * c);
    }
    return w;
}

enum GenKind : int { GEN_GRAY = 0, GEN_RANDOM = 1, GEN_PERTURB = 2, GEN_EXPLICIT = 3,
                     GEN_SYM = 4 };   // internal: exhaustive GRAY, one placement per relabelling class

// Restricted-growth-string completion counts for GEN_SYM (search_kernel.cuh
// RgsGen): rgs[M][rem·kRgsStride + m], m = devices in use (1..M).
constexpr int kRgsStride = 9;
constexpr int kRgsRows = 65;

constexpr uint64_t kInfeasible = ~0ull;
constexpr int kMaxImageBytes = 96 * 1024;
constexpr int kMaxSmemBytes = 227 * 1024;
constexpr int kTierSmemBytes = 200 * 1024;   // shared-memory tier: image + 4 warps of lane state

// Kernel parameters (by value).
struct KParams {
    const uint8_t *g_image;      // device image (16-B aligned, padded)
    const uint8_t *g_place;      // explicit placements [count][K] (device)
    uint64_t *g_makespan;        // write-all output [end-begin]
    uint64_t *g_partials;        // [grid][2] per-CTA argmin
    unsigned *g_ticket;          // last-CTA counter (self-resetting)
    uint64_t *g_out;             // {makespan, index}
    uint64_t begin, end;         // candidate range
    uint64_t seed;               // seed of this round (RANDOM/PERTURB)
    uint64_t cap;                // memory cap (0 = none)
    uint32_t image_bytes;
    uint32_t K, K8;
    uint32_t off_extra, off_mem, off_orig;
    uint32_t tau;
    uint32_t smem_slots_off;     // byte offset of the first warp region in smem
    uint32_t region_bytes;       // bytes per warp region
    uint32_t free_off;           // region offset of free[M] (M ≥ 3), in slot units ×256
    uint32_t zero_off;           // region offset of the always-zero slot, in slot units ×256
    uint32_t one_hi;             // 0x3FF00000, the high word of 1.0 (opaque to ptxas)
    uint32_t off_cls;            // hardware graph: image offset of cls[a·8 + b]
    uint32_t off_hgw;            // image offset of the half-group base words (u32 × K8/4)
    const uint64_t *g_rgs;       // GEN_SYM: RGS completion counts of this M (device)
    unsigned long long *g_tile;  // argmin kernels: next tile (dynamic, reset by the last CTA)
    uint8_t *g_state;            // global-state tier: warp regions of the lane state (search_big_kernel)
};

// ---- exact-schedule image, built when
// N = 2K ≤ 64 nodes:
//   [XNode × N]        node n < K: forward of π position n; n ≥ K: backward of
//                      π position n − K.  N-node order F_0..F_{K−1},
//                      B_{K−1}..B_0 is topological.
//   [XPred × NA]       predecessor arcs, contiguous per node
//   [u64 × nrows·xcls] arc cost (ps) per device-pair class; row 0 is all zero
//                      (the F_p → B_p arc and zero-cost inputs)
//   [u8 × 64]          class of the ordered device pair (a, b), 0 iff a = b
//   [u64 × K]          M(k) by π position
//   [u8 × K]           descriptor index of π position p
struct XNode {
    uint64_t dur;         // Δf or Δb
    uint64_t tail0;       // longest path from the node to the end with zero communication
    uint64_t predmask;    // bit q set iff node q is a predecessor
    uint16_t pred_begin;  // first XPred
    uint8_t npred;        // number of XPred
    uint8_t pos;          // π position (its device is the placement's device of pos)
    uint32_t pad;
};
static_assert(sizeof(XNode) == 32, "XNode is 32 B");
struct XPred {
    uint8_t node;         // predecessor node
    uint8_t pad;
    uint16_t row;         // cost row
};
constexpr int kMaxExactNodes = 64;

// ---- EFT image, any K:
//   [GOp × K]          forward op of π position p
//   [GArc × NA]        its forward in-arcs
//   [u64 × nrows·gcls] cost rows (as in the exact image; row 0 all zero)
//   [u8 × 64]          class of the ordered device pair
struct GOp {
    uint64_t fwd;         // Δf
    uint64_t mem;         // M(k)
    uint32_t in_begin, in_cnt;
    uint64_t pad;
};
static_assert(sizeof(GOp) == 32, "GOp is 32 B");
struct GArc {
    uint32_t u;           // producer's π position
    uint32_t row;         // cost row
};

// ---- pipeline-parallel MP, built on first use:
// π-prefix sums of Δf, Δb, M(k) ([K+1] each), 2-D prefix sums over
// (producer π position, consumer π position) of the edges' forward bytes,
// backward bytes and count ([(K+1)²] each), binomials C(n, k) for k < 8.
struct PipeParams {
    const uint64_t *g_pf, *g_pb, *g_pm, *g_qf, *g_qb, *g_qc, *g_binom;
    uint64_t *g_makespan;        // optional per-candidate output [end − begin]
    uint64_t *g_partials;        // [grid][2]
    unsigned *g_ticket;
    uint64_t *g_out;             // {makespan, index} or null
    uint64_t bw, lat, cap, begin, end, block;
    uint64_t overhead;           // per op per micro-batch (ps)
    uint32_t K, nm;
    uint32_t micro[16];
};
constexpr int kMaxPipelineK = 1024;
int launch_pipeline(int M, const PipeParams &p, int grid, void *stream);
int pipeline_block_threads(int M);   // 256, or 128 when M ≥ 5 (pair columns in shared memory)

// per-warp branch-and-bound state of the exact kernel (shared memory)
struct XWarp {
    uint64_t fin[kMaxExactNodes];
    uint64_t cand[kMaxExactNodes + 1];
    uint64_t oldfree[kMaxExactNodes + 1];
    uint64_t oldpm[kMaxExactNodes + 1];
    uint64_t head[kMaxExactNodes];     // longest path to the node's start (this placement's delays)
    uint64_t tail[kMaxExactNodes];     // longest path from the node's start to the end
    uint64_t ebuf[kMaxExactNodes];     // per-expand lower bound on each unscheduled node's start
    uint64_t freeT[8];
    uint64_t rem[8];
    uint8_t chosen[kMaxExactNodes + 1];
    uint8_t ystar[kMaxExactNodes + 1];
    uint8_t dev[kMaxExactNodes];       // by π position
    uint8_t pad[14];
};

struct XParams {
    const uint8_t *g_ximage;
    const uint8_t *g_place;      // explicit placements [count][K] (descriptor order)
    const uint8_t *g_base;       // PERTURB base, π order
    uint64_t *g_makespan;        // per-candidate output [end − begin] (or null in search mode)
    uint8_t *g_exact;            // per-candidate 1 = exact, 0 = node limit hit (optional)
    uint64_t *g_partials;        // search mode: [grid][2] per-CTA argmin
    unsigned *g_ticket;
    uint64_t *g_out;             // search mode: {makespan, index, unresolved}
    unsigned long long *g_work;  // [0] next candidate, [1] incumbent makespan, [2] unresolved count
    uint64_t begin, end, seed, cap, node_limit;
    uint32_t x_bytes, N, K, xcls, tau;
    uint32_t off_pred, off_rows, off_cls, off_mem, off_orig;
    uint32_t ws_off;             // smem offset of the first per-warp state block
    int search;                  // 1: argmin with incumbent pruning
    const uint64_t *g_rgs;       // GEN_SYM: RGS completion counts of this M (device)
};
typedef int (*XLaunchFn)(const XParams &, int grid, int threads, int smem, void *stream);
struct XKernelInfo {
    XLaunchFn launch;
    const void *func;
};
XKernelInfo exact_kernel_for(int M, int gen);

// Device scalar slots of pp_dfg::d_scalars (u64).
enum ScalarSlot : int {
    SC_LOCAL_MK = 0, SC_LOCAL_IDX = 1,       // this GPU's argmin of the round
    SC_KEY_LOCAL = 2, SC_KEY_GLOBAL = 3,     // packed key, before / after min all-reduce
    SC_IDX_LOCAL = 4, SC_IDX_GLOBAL = 5,     // winner-index contribution / result
    SC_BEST_MK = 6, SC_BEST_IDX = 7, SC_BEST_ROUND = 8,
    SC_COUNT = 16
};
static_assert(SC_LOCAL_MK == proto::LOCAL_MK && SC_LOCAL_IDX == proto::LOCAL_IDX && SC_KEY_LOCAL == proto::KEY_LOCAL &&
                  SC_KEY_GLOBAL == proto::KEY_GLOBAL && SC_IDX_LOCAL == proto::IDX_LOCAL &&
                  SC_IDX_GLOBAL == proto::IDX_GLOBAL,
              "scalar slots follow protocol.h");

struct UParams {
    uint8_t *image;       // device image: the PERTURB base is patched into OpRec.base
    uint8_t *base;        // PERTURB base, π order (device)
    uint8_t *winner;      // scratch [K]
    uint8_t *best_place;  // [K] best placement so far, π order
    uint64_t *s;          // d_scalars
    uint64_t seed;        // seed of this round
    uint32_t K, K8, tau, round;
    int multi;            // 1: winner comes from the NCCL-reduced slots
    uint32_t off_hgw;     // image offset of the half-group base words
};
typedef int (*UpdateFn)(const UParams &, void *stream);

// Launch one search/eval kernel instantiation. Returns a cudaError_t value.
// threads: CTA size; grid: number of CTAs; smem: dynamic shared bytes.
typedef int (*LaunchFn)(const KParams &, int grid, int threads, int smem, void *stream);

struct KernelInfo {
    LaunchFn launch;
    const void *func;            // for occupancy queries / attributes
};

// search_inst.cu (compiled once per M with -DPP_M): kernel_for_m<M>(...)
KernelInfo kernel_for(int M, int gen, bool mem, bool write_all, bool f64, int np, bool hw);
// the global-state tier: one kernel per (M, generator, arithmetic), big_np(M)
// placements per lane
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr int big_np(int M) { return M <= 2 ? 2 : 1; }
KernelInfo big_kernel_for(int M, int gen, bool f64);
UpdateFn update_for(int M, int gen);

}  // namespace pp

struct pp_dfg {
    int device = 0;
    int K = 0, K8 = 0, E = 0, W = 0;
    bool f64 = false;            // tagged-f64 arithmetic (bound < 2^49) else tagged-u64
    bool hw = false;             // general hardware graph: class-cost rows (pp_load_dfg_hw)
    bool big = false;            // global-state tier: image or lane state beyond shared memory
    int nd = 0;                  // hardware-graph devices
    uint32_t off_cls = 0;        // image offset of the 8×8 class table
    uint64_t t1 = 0, grad_bytes = 0, cap = 0;
    std::vector<int32_t> pi;     // π position → descriptor index
    std::vector<int32_t> pos;    // descriptor index → π position
    std::vector<uint64_t> param; // param_bytes by descriptor index
    uint64_t link_bw = 0, link_lat = 0;            // uniform link (0 in hw mode)
    std::vector<int32_t> e_src, e_dst;             // edges by π position
    std::vector<uint64_t> e_bf, e_bb, fwd, bwd, mem;   // bytes; Δf, Δb, M(k) by π position
    uint64_t *d_pipe = nullptr;                    // pipeline tables (lazily built)
    mutable uint64_t *d_rgs = nullptr;             // RGS completion counts, every M (lazily built)
    mutable std::map<int, int> tuned;              // (M, gen) -> measured best NP
    std::vector<uint8_t> image;  // host copy of the image
    uint32_t off_extra = 0, off_mem = 0, off_orig = 0, off_hgw = 0, image_bytes = 0;
    uint32_t base_bytes = 0;     // K rounded up to 16
    // exact-schedule image (empty when 2K > 64)
    std::vector<uint8_t> ximage;
    uint32_t xN = 0, xcls = 0, x_bytes = 0;
    uint32_t x_off_pred = 0, x_off_rows = 0, x_off_cls = 0, x_off_mem = 0, x_off_orig = 0;
    uint8_t *d_ximage = nullptr;
    // EFT image
    std::vector<uint8_t> gimage;
    uint32_t g_off_arc = 0, g_off_rows = 0, g_off_cls = 0, g_bytes = 0, gcls = 0;
    uint8_t *d_gimage = nullptr;
    unsigned long long *d_xwork = nullptr;   // [4]
    // device memory
    uint8_t *d_image = nullptr;
    uint8_t *d_base = nullptr;        // [base_bytes] PERTURB base (π order)
    uint8_t *d_winner = nullptr;      // [base_bytes] scratch placement
    uint8_t *d_best_place = nullptr;  // [base_bytes]
    uint64_t *d_partials = nullptr;   // [kMaxGrid][2]
    unsigned *d_ticket = nullptr;
    uint64_t *d_scalars = nullptr;    // see capi.cpp (round result, keys, best)
    int sm_count = 0;
    uint8_t *d_state = nullptr;       // global-state tier scratch (grown on demand)
    size_t state_bytes = 0;
};

namespace pp {
void set_error(const std::string &msg);
void note_launch();
constexpr int kMaxGrid = 148 * 32;
}
