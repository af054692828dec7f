/*
 * pp.h — C ABI of the B200-native placement-evaluation / hybrid-projection
 * library (libpp.so), the data-parallel hot path of arXiv 1907.13257
 * "Optimizing Multi-GPU Parallelization Strategies for Deep Learning Training".
 *
 * Citations are line numbers of /root/reference/PAPER.md (and SPEC.md) with
 * the section / equation they fall in; the readings R1–R20 are listed in
 * DESIGN.md §Readings.
 *
 * Conventions for every entry point
 *   - Return value: PP_OK (0) or a negative PP_E_* code; pp_last_error()
 *     then returns a thread-local message describing the failure.
 *   - "host ptr": caller-owned host memory, read (or written) during the call
 *     only, never retained.  "device ptr": caller-owned device memory on the
 *     pp_dfg's CUDA device (e.g. torch tensor .data_ptr()), accessed in
 *     stream order on `cuda_stream` (a cudaStream_t; NULL = legacy default
 *     stream).  Nothing is freed across the boundary.
 *   - Handles (pp_dfg, pp_comm) are library-owned; release them with
 *     pp_free_dfg / pp_comm_destroy.  Calls on one pp_dfg must not overlap
 *     in time (they share its device scratch); distinct pp_dfg are
 *     independent.
 *   - Times are integer picoseconds (u64), bytes are u64, bandwidths are
 *     bytes per second.  All results are exact integers (no floating point).
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     entry point fails with PP_E_CUDA.
 */
#ifndef PP_H
#define PP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PP_OK            0
#define PP_E_INVALID    (-1) /* bad argument, M outside [1,8], self edge, dangling
                                endpoint, duplicate/negative id      */
#define PP_E_CYCLE      (-2) /* the DFG has a cycle; message names one cycle's ids  */
#define PP_E_RANGE      (-3) /* a time bound ≥ 2^61 ps or a u128 product overflow   */
#define PP_E_TOO_LARGE  (-4) /* GRAY space M^K > 2^63; K > 65535, W + 1 > 4096 or
                                an image ≥ 2 GB; a hardware graph beyond the
                                shared-memory tier (pp_dfg_get_tier)                */
#define PP_E_INFEASIBLE (-5) /* every evaluated candidate violates device memory    */
#define PP_E_CUDA       (-6) /* CUDA failure or no device                           */
#define PP_E_NCCL       (-7) /* NCCL unavailable or failed                          */

#define PP_INFEASIBLE_MAKESPAN UINT64_MAX /* makespan of a memory-infeasible placement */

typedef struct pp_dfg pp_dfg;   /* opaque: a DFG resident on one GPU            */
typedef struct pp_comm pp_comm; /* opaque: an NCCL communicator (one per rank)  */

/* ------------------------------------------------------------------ DFG --
 * The compute DFG of PAPER.md:350 (§6, Table 2): vertices K
 * with expected execution time Δ(k) and memory footprint M(k); directed edges
 * E with D(e) bytes.  Reading R1: each op has a forward time Δf and a backward
 * time Δb; the backward op runs on the forward op's device and every edge
 * carries activation bytes forward and gradient bytes backward.
 * Arrays are indexed by descriptor index k = 0..num_ops-1 (ops) and
 * e = 0..num_edges-1 (edges); all are host ptrs copied by pp_load_dfg.      */
typedef struct {
    int32_t         num_ops;        /* K ≥ 1                                        */
    int32_t         num_edges;      /* E ≥ 0; parallel edges allowed   */
    const int64_t  *op_id;          /* [K] external ids ≥ 0, unique; NULL ⇒ k.  The
                                       topological order π is Kahn's algorithm with
                                       ties to the smallest id (R3)   */
    const uint64_t *fwd_ps;         /* [K] Δf(k) ps                   */
    const uint64_t *bwd_ps;         /* [K] Δb(k) ps (R1)                             */
    const uint64_t *mem_bytes;      /* [K] M(k); NULL ⇒ 0            */
    const uint64_t *param_bytes;    /* [K] weight bytes; S_grad = Σ; NULL ⇒ 0        */
    const int32_t  *edge_src;       /* [E] descriptor index of the producer          */
    const int32_t  *edge_dst;       /* [E] descriptor index of the consumer (≠ src)  */
    const uint64_t *edge_fwd_bytes; /* [E] D(e) activation bytes      */
    const uint64_t *edge_bwd_bytes; /* [E] gradient bytes; NULL ⇒ = edge_fwd_bytes  */
} pp_dfg_desc;

/* The hardware graph of PAPER.md:352 reduced to M identical devices behind
 * one NVSwitch hop (R4): a cut edge costs c(e) = ⌈D(e)·10^12 / BW⌉ + L ps
 * (Δ_e = Σ_l C_el·(D(e)/B(l)+L(l)), one hop).            */
typedef struct {
    uint64_t link_bw_Bps;        /* B(l) > 0                                        */
    uint64_t link_lat_ps;        /* L(l)                                            */
    uint64_t dev_mem_cap_bytes;  /* Mem(n); 0 = unlimited (R7)   */
} pp_link_desc;

/* The general hardware graph (Table 2
 * PAPER.md:379–392): device nodes 0..num_devices−1, router nodes
 * num_devices..num_devices+num_routers−1, bidirectional links with bandwidth
 * B(l) > 0 B/s and latency L(l) ps.  A cut edge e from device a to device b
 * costs the delay of its delay-shortest route for its payload
 * (PAPER.md:455–462 Δ_e = Σ_l C_el·(D(e)/B(l) + L(l))):
 *   c(e, a, b) = min over paths a → b of Σ_hops (⌈D(e)·10^12 / B⌉ + L).
 * A search with M devices uses devices 0..M−1 (M ≤ num_devices).            */
typedef struct {
    int32_t         num_devices;      /* 1..8                                       */
    int32_t         num_routers;      /* ≥ 0                                        */
    int32_t         num_links;
    const int32_t  *link_a, *link_b;  /* [num_links] node ids, a ≠ b                 */
    const uint64_t *link_bw_Bps;      /* [num_links] B(l) > 0                        */
    const uint64_t *link_lat_ps;      /* [num_links] L(l)                            */
    uint64_t        dev_mem_cap_bytes;/* Mem(n), 0 = unlimited                        */
} pp_hw_desc;

typedef struct {
    int32_t  num_ops, num_edges;
    int32_t  num_slots;          /* W: live finish-time slots per placement         */
    int32_t  image_bytes;        /* shared-memory image size                        */
    uint64_t t1_ps;              /* T_1 = Σ_k (Δf+Δb): all ops on one device (R8)   */
    uint64_t grad_bytes;         /* Σ param_bytes                                   */
} pp_dfg_info;

/* Validates the DFG, builds π, the per-edge ps costs, the forward+backward
 * schedule records and the liveness slots, and uploads the packed image to
 * `cuda_device`.  Errors: PP_E_INVALID, PP_E_CYCLE (message lists the ids of
 * one cycle), PP_E_RANGE (Σ(Δf+Δb) + Σ(c_f+c_b) ≥ 2^61), PP_E_TOO_LARGE,
 * PP_E_CUDA.  On success *out owns device memory until pp_free_dfg.         */
int  pp_load_dfg(const pp_dfg_desc *desc, const pp_link_desc *link, int cuda_device,
                 pp_dfg **out);
/* As pp_load_dfg on a general hardware graph.  Device pairs whose cost on
 * every edge (both directions) agree share a cost class; the image holds one
 * cost row per input and class.  Needs every time bound < 2^49 ps (tagged-f64
 * arithmetic) else PP_E_RANGE; devices must be connected else PP_E_INVALID;
 * PP_E_TOO_LARGE when the rows do not fit in the 96 KB image.              */
int  pp_load_dfg_hw(const pp_dfg_desc *desc, const pp_hw_desc *hw, int cuda_device, pp_dfg **out);
void pp_free_dfg(pp_dfg *dfg);
/* Host only (no CUDA device needed): what pp_load_dfg would build for this
 * DFG — validation with the same errors, π, the slot allocation (num_slots =
 * W), the image size, T_1, Σ param_bytes — and the state tier it would run on
 * (*tier = PP_TIER_SHARED / PP_TIER_GLOBAL, pp_dfg_get_tier).  Host ptrs.   */
int  pp_plan_dfg(const pp_dfg_desc *desc, const pp_link_desc *link, pp_dfg_info *info, int32_t *tier);
int  pp_dfg_get_info(const pp_dfg *dfg, pp_dfg_info *out);
/* The state tier the DFG runs on, decided at load time:
 *   PP_TIER_SHARED  image and lane state in shared memory (every kernel);
 *   PP_TIER_GLOBAL  the image (> 96 KB) or the per-lane state ((W + 1 + M)
 *                   slots × 8 B; fewer than 4 resident warps per SM would fit)
 *                   beyond shared memory: the search/eval calls run
 *                   search_big_kernel (image read from HBM through L1/L2, lane
 *                   state in a global scratch, tagged-u64 arithmetic) with
 *                   identical results.  The symmetry-reduced exhaustive search
 *                   is not used there (the plain Gray order gives the same
 *                   argmin); hardware graphs are rejected (PP_E_TOO_LARGE).
 * The environment variable PP_TIER=global, read by pp_load_dfg, forces the
 * global tier (tests).  Returns the tier, or PP_E_INVALID for NULL.         */
#define PP_TIER_SHARED 0
#define PP_TIER_GLOBAL 1
int  pp_dfg_get_tier(const pp_dfg *dfg);
/* host ptr pi_out[K]: pi_out[p] = descriptor index of the op at π position p */
int  pp_dfg_get_pi(const pp_dfg *dfg, int32_t *pi_out);

/* ------------------------------------------------- placement evaluation --
 * Step makespan of explicit placements (P_kn of PAPER.md:396, Σ_n P_kn = 1 of
 * PAPER.md:414–421): forward ops in π order then backward ops in reverse π
 * order, each op starting at max(data ready, device free) (PAPER.md:443–453
 * dependency, :465–476 non-overlap, :497–503 assumptions; R1, R2).
 *   d_placements : device ptr uint8 [count][K], row i = candidate i, column k =
 *                  device of descriptor op k, each < M
 *   d_makespan   : device ptr uint64 [count]; PP_INFEASIBLE_MAKESPAN when the
 *                  memory cap is violated
 * Asynchronous on cuda_stream.  A row holding a value ≥ M is not an error
 * of the call: the device checks every value, evaluates nothing out of range,
 * and writes PP_INFEASIBLE_MAKESPAN for that row; other rows are unaffected. */
int pp_eval_placements(const pp_dfg *dfg, int M, const uint8_t *d_placements, uint64_t count,
                       uint64_t *d_makespan, void *cuda_stream);

/* Candidate generators (the paper has no generator):
 *   GRAY    reflected M-ary Gray code of the candidate index over π positions;
 *           index 0 = all on device 0; count ≤ M^K ≤ 2^63 (= M^K: exhaustive)
 *   RANDOM  SplitMix64 words, b = ⌈log2 M⌉ bits per op; index 0 = all zero
 *   PERTURB per op flip with probability flip_thresh/256: M = 2 to the other
 *           device, M = 4, 8 re-drawn uniformly (base ⊕ y, y mod M), other M
 *           to one of the other M−1 devices (generator revision 3, DESIGN.md
 *           §2); index 0 = the base; round r uses seed+r
 * Exhaustive GRAY (the whole range [0, M^K), uniform link, M ≥ 2, K ≥ 2) is
 * evaluated one placement per device-relabelling class, with the oracle's
 * (makespan, Gray index) winner; the
 * results are those of the full enumeration (PP_NO_SYM=1 runs it unreduced). */
typedef enum { PP_GEN_GRAY = 0, PP_GEN_RANDOM = 1, PP_GEN_PERTURB = 2 } pp_gen;

typedef struct {
    int32_t        gen;          /* pp_gen                                           */
    uint32_t       rounds;       /* ≥ 1; > 1 only for PERTURB                        */
    uint64_t       seed;
    uint64_t       count;        /* candidates per round, ≥ 1                        */
    uint32_t       flip_thresh;  /* PERTURB τ ∈ [0, 256]                             */
    uint32_t       _pad;
    const uint8_t *base;         /* host ptr [K] descriptor order; NULL ⇒ all zero  */
} pp_search_desc;

typedef struct {
    uint64_t best_makespan_ps;   /* T_M: the best makespan found                     */
    uint64_t best_index;         /* its candidate index within best_round            */
    uint64_t best_round;         /* first round that reached best_makespan_ps        */
    uint64_t t1_ps;              /* T_1; SU_MP(M) = t1_ps / best_makespan_ps
                                    (§3.2)                         */
    uint64_t evaluated;          /* count × rounds over all ranks                    */
    uint8_t *placement;          /* host ptr [K] caller-owned, filled in descriptor
                                    order; may be NULL                               */
} pp_search_result;

/* Makespans of generated candidates begin..begin+count-1 of one round (seed_r
 * already includes the round offset).  d_base: device ptr uint8 [K] in π
 * order (PERTURB only, else may be NULL).  d_makespan: device ptr [count].  */
int pp_eval_generated(const pp_dfg *dfg, int M, int gen, uint64_t seed_r, uint32_t flip_thresh,
                      const uint8_t *d_base_pi, uint64_t begin, uint64_t count,
                      uint64_t *d_makespan, void *cuda_stream);

/* The lexicographically smallest (makespan, index) over candidates
 * [begin, end) of one round, computed on the GPU (in-warp shuffle, CTA and
 * grid argmin).  d_best: device ptr uint64[2] = {makespan, index}.          */
int pp_search_range(const pp_dfg *dfg, int M, int gen, uint64_t seed_r, uint32_t flip_thresh,
                    const uint8_t *d_base_pi, uint64_t begin, uint64_t end, uint64_t *d_best,
                    void *cuda_stream);

/* ------------------------------------------- exact schedule (§8(f) f1) --
 * The makespan-OPTIMAL schedule of each placement instead of the in-order
 * list schedule: DLPlacer "minimizes per step training time by ...
 * determining the execution start time of each vertex on a device"
 * (§6) under the dependency and non-overlap
 * constraints; SPEC.md:161–169 exact_schedule.  Per-device
 * execution order is free (reading R22); the result is ≤ the
 * in-order makespan of the same placement.  Branch and bound on the GPU, one
 * warp per placement; exponential in the worst case, so it needs
 * 2K ≤ 64 nodes (K ≤ 32 ops) else PP_E_TOO_LARGE.
 *   node_limit   branch-and-bound nodes per placement before giving up
 *                (0 ⇒ 2^24).  A placement that hits it gets the best
 *                makespan found so far (an upper bound) and d_exact[i] = 0.
 *   d_exact      device ptr uint8 [count], optional (NULL): 1 = optimal.
 * Placements and generators as in pp_eval_placements / pp_eval_generated;
 * memory-infeasible placements, and explicit rows holding a value ≥ M, give
 * PP_INFEASIBLE_MAKESPAN.  Asynchronous.                                    */
int pp_eval_exact(const pp_dfg *dfg, int M, const uint8_t *d_placements, uint64_t count,
                  uint64_t node_limit, uint64_t *d_makespan, uint8_t *d_exact, void *cuda_stream);
int pp_eval_exact_generated(const pp_dfg *dfg, int M, int gen, uint64_t seed_r, uint32_t flip_thresh,
                            const uint8_t *d_base_pi, uint64_t begin, uint64_t count, uint64_t node_limit,
                            uint64_t *d_makespan, uint8_t *d_exact, void *cuda_stream);
/* Lexicographically smallest (exact makespan, index) over candidates
 * [begin, end) of one round.  Placements whose bound already exceeds the
 * best makespan found so far are abandoned early (they cannot win); the
 * incumbent starts at the in-order argmin of the same candidates, an upper
 * bound of the exact optimum (each placement's exact makespan ≤ its
 * in-order one), so ties at the optimum are never pruned.
 * d_best: device ptr uint64[3] = {makespan, index, number of placements that
 * hit node_limit (0 ⇒ the result is exact)}.  Asynchronous.                 */
int pp_search_exact(const pp_dfg *dfg, int M, int gen, uint64_t seed_r, uint32_t flip_thresh,
                    const uint8_t *d_base_pi, uint64_t begin, uint64_t end, uint64_t node_limit,
                    uint64_t *d_best, void *cuda_stream);

/* ----------------------------------- pipeline-parallel MP (§8(f) f3) --
 * GPipe-style pipelining (§2; §4.4: how GNMT and
 * BigLSTM were split).  Reading R26: M stages are contiguous
 * π ranges [cut_s, cut_{s+1}) on devices 0..M−1; a mini-batch is split into m
 * micro-batches, stage times ⌈ΣΔ/m⌉ + n_s·overhead_ps (n_s ops in the stage; a
 * fixed per-op cost every micro-batch pays — the "kernel overheads" of
 * PAPER.md:299, reading R27; 0 = none); the activations of a micro-batch from
 * stage a to b travel as one transfer ⌈D_ab·10^12/(m·BW)⌉ + L (uniform link);
 * forward micro-batches in order, then the backward in reverse order; the
 * makespan is the last stage's finish.  Candidates: index = rank·nm + j, rank
 * = lexicographic rank of the cut vector (C(K−1, M−1) of them), j indexes
 * micro[] (nm ≤ 16).  Needs K ≤ 1024 and a uniform-link pp_dfg.            */
typedef struct {
    uint64_t makespan_ps;        /* T_M of the best pipeline (SU = T_1 / T_M)   */
    uint64_t index;              /* its candidate index                         */
    uint64_t candidates;         /* C(K−1, M−1)·nm                              */
    uint32_t micro_batches, n_stages;
    int32_t  cuts[8];            /* first π position of stages 1..M−1          */
} pp_pipeline_result;

/* *count = C(K−1, M−1)·nm (PP_E_TOO_LARGE if ≥ 2^63). */
int pp_pipeline_space(const pp_dfg *dfg, int M, int nm, uint64_t *count);
/* Candidates [begin, end): d_best (device ptr uint64[2] = {makespan, index},
 * lexicographic argmin) and/or d_makespan (device ptr uint64 [end−begin]).
 * micro: host ptr uint32 [nm].  Asynchronous.                               */
int pp_pipeline_range(const pp_dfg *dfg, int M, const uint32_t *micro, int nm, uint64_t overhead_ps,
                      uint64_t begin, uint64_t end, uint64_t *d_best, uint64_t *d_makespan, void *cuda_stream);
/* The whole space; fills *out (host ptr) with the winner's cuts.
 * Synchronises cuda_stream.  PP_E_INFEASIBLE if every stage split violates
 * the memory cap.                                                           */
int pp_pipeline_search(const pp_dfg *dfg, int M, const uint32_t *micro, int nm, uint64_t overhead_ps,
                       void *cuda_stream, pp_pipeline_result *out);

/* ----------------------------------------- EFT base seed (§8(f) f4) --
 * The earliest-finish-time greedy placement (SPEC.md:245–253
 * heuristic_place; reading R23): forward ops in π order, each
 * on the device where it would finish first given the ops already placed and
 * the incoming transfer delays (ties → smaller device), skipping devices
 * whose memory would exceed the cap.  A good PERTURB base
 * (pp_search_desc.base).  placement: host ptr uint8 [K], descriptor order.
 * Synchronises cuda_stream.  Errors: PP_E_INVALID, PP_E_INFEASIBLE (an op
 * fits on no device), PP_E_CUDA.                                            */
int pp_eft_place(const pp_dfg *dfg, int M, uint8_t *placement, void *cuda_stream);

/* Full search: per round the candidates are sharded over
 * the ranks of `comm` (contiguous slices, see pp_rank_slice), each GPU takes
 * its slice's argmin, one NCCL min all-reduce of the packed key
 * (pp_pack_key) gives the winning makespan, a second min all-reduce delivers
 * the smallest index reaching it (pp_round_contrib); PERTURB moves the base to the round winner when it is
 * strictly better.  comm = NULL: single GPU.  The result is identical for any
 * number of ranks.  Synchronises cuda_stream before returning.
 * Errors: PP_E_INVALID, PP_E_TOO_LARGE (GRAY space), PP_E_INFEASIBLE,
 * PP_E_CUDA, PP_E_NCCL.                                                      */
int pp_search_best(const pp_dfg *dfg, int M, const pp_search_desc *desc, pp_comm *comm,
                   void *cuda_stream, pp_search_result *out);

/* ------------------------------------------------------------ multi-GPU --
 * NCCL is loaded at run time (dlopen "libnccl.so.2", normally the copy torch
 * already loaded).  The unique id is 128 bytes (ncclUniqueId) and is passed
 * between processes by the caller (e.g. a torch.distributed broadcast).     */
int  pp_comm_get_unique_id(uint8_t out_id[128]);
int  pp_comm_init(const uint8_t id[128], int rank, int world, int cuda_device, pp_comm **out);
void pp_comm_destroy(pp_comm *comm);

/* The (makespan, index) argmin across the ranks of comm:
 * each rank's d_best (device ptr uint64[2] = {makespan, index} over its own
 * candidate slice, e.g. from pp_search_range / pp_search_exact /
 * pp_pipeline_range on its pp_rank_slice; {PP_INFEASIBLE_MAKESPAN, UINT64_MAX}
 * for an empty slice) is replaced in place by the global lexicographic
 * argmin: one NCCL min all-reduce of the packed key (pp_round_key: the
 * smallest makespan, ties to the lowest rank, i.e. the lowest indices for
 * contiguous slices; an empty slice never wins), a second of the winner's
 * index — the same exchange pp_search_best runs every round.
 * Synchronises cuda_stream, polling the communicator for asynchronous NCCL
 * errors and the comm's timeout (pp_comm_set_timeout) while it waits; on an
 * error or a timeout the communicator is aborted and PP_E_NCCL returned (the
 * comm is then unusable; destroy it).  Errors: PP_E_INVALID, PP_E_NCCL,
 * PP_E_CUDA.                                                                 */
int pp_argmin_allreduce(const pp_dfg *dfg, pp_comm *comm, uint64_t *d_best, void *cuda_stream);

/* Timeout for the waits of pp_search_best / pp_argmin_allreduce on this comm
 * (a dead or stalled rank otherwise hangs the collective).  0 ⇒ the default,
 * PP_NCCL_TIMEOUT_S from the environment or 600 s.                          */
int pp_comm_set_timeout(pp_comm *comm, uint64_t timeout_ms);

/* Sharding protocol (host only, no GPU needed).  These are the functions the
 * device kernels and the NCCL driver run (csrc/protocol.h), exported so that
 * multi-process CPU tests exercise the product's own rules and sequence:
 *   rank r of R owns candidates [⌊r·n/R⌋, ⌊(r+1)·n/R⌋) of every round;
 *   key = (min(makespan, 2^61−1) << 3) | r for a slice whose local argmin
 *   index is not UINT64_MAX, else UINT64_MAX (an empty slice never wins), R ≤ 8;
 *   the minimum key carries the winning makespan; every rank whose key has
 *   that makespan contributes its local argmin index, every other rank
 *   UINT64_MAX, to a second min all-reduce, so the result is the smallest
 *   global index with the minimum makespan for any slice layout.            */
void     pp_rank_slice(uint64_t count, int rank, int world, uint64_t *begin, uint64_t *end);
uint64_t pp_round_key(uint64_t makespan, uint64_t index, int rank);
uint64_t pp_pack_key(uint64_t makespan, int rank);   /* = pp_round_key(makespan, 0, rank) */
uint64_t pp_key_makespan(uint64_t key);   /* 2^61−1 (and UINT64_MAX) map back to PP_INFEASIBLE_MAKESPAN */
int      pp_key_rank(uint64_t key);
uint64_t pp_round_contrib(uint64_t key_global, uint64_t key_local, uint64_t local_index);
/* 1 iff a PERTURB base moves to the round winner with this global index (the
 * winner is strictly better than the base exactly when it is not candidate 0) */
int      pp_round_moves_base(uint64_t win_index);
/* One round's exchange on the host with a caller-supplied collective:
 * allreduce_min(ctx, in, out) must set *out to the minimum of `in` over all
 * ranks (0 = success).  The sequence is the one the NCCL path runs.
 * win[0] = winning makespan (PP_INFEASIBLE_MAKESPAN if none), win[1] = index. */
typedef int (*pp_allreduce_min_u64)(void *ctx, uint64_t in, uint64_t *out);
int pp_round_exchange_host(uint64_t local_makespan, uint64_t local_index, int rank,
                           pp_allreduce_min_u64 allreduce_min, void *ctx, uint64_t win[2]);

/* ------------------------------------------------------------ projection --
 * End-to-end training time C = T × S × E (Eq. 1) for DP-only
 * (M = 1) and hybrid M-way MP × W-way DP (Eq. 5) at every
 * device count N = 1..N_max (SURVEY.md §8(c) O8–O10):
 *   W = N/M workers (cell infeasible when M ∤ N, R15), G = W·B,
 *   S = ⌈D/G⌉ (R14), E = E(G) from the knots (linear in G with
 *   floor, infeasible outside the knots, R12),
 *   AR(W) = 0 if W = 1 else ⌈2(W−1)·S_grad·10^12/(W·BW)⌉ + 2(W−1)·α with the
 *   intra tier if N ≤ node_size else the inter tier (R10;
 *   a tier with BW = 0 is "SE ≡ 1"),
 *   T = ⌊(T_1 + AR)·T_M / T_1⌋ (EQ5, SU^M·SE_W of Eq. 5, R11) or T_M + AR (TIME).
 * Gradient-accumulation axis (PAPER.md:251 delayed
 * gradient update; R25): with factors a ∈ accum[], a cell accumulates a
 * mini-batches per step: G = W·B·a, T = ⌊(a·T_1 + AR)·T_M / T_1⌋ (EQ5) or
 * a·T_M + AR (TIME); the cell keeps the a with the least C (ties → earlier in
 * accum[]) in pp_cell.accum.  Placement-aware all-reduce (R24): with
 * shard_bytes, hybrid M all-reduces each device's shard over its W peers in
 * parallel, AR = max_d AR(W, S_d) (pp_shard_bytes gives S_d of a placement). */
typedef struct {
    uint64_t        dataset_items;   /* D ≥ 1                                   */
    uint32_t        mini_batch;      /* B ≥ 1                                   */
    uint32_t        n_knots;         /* ≥ 1                                     */
    const uint64_t *knot_G;          /* host ptr [n_knots], strictly increasing */
    const uint64_t *knot_uepochs;    /* host ptr [n_knots], µ-epochs, > 0       */
    uint64_t        grad_bytes;      /* S_grad                                  */
    uint64_t        bw_intra_Bps, lat_intra_ps, bw_inter_Bps, lat_inter_ps;
    uint32_t        node_size;       /* 0 ⇒ 8                                   */
    uint32_t        ar_mode;         /* 0 = EQ5 (default), 1 = TIME             */
    uint64_t        t1_ps;           /* T_1 > 0                                 */
    uint32_t        n_accum;         /* 0 ⇒ a = 1 only; else ≤ 32 factors       */
    uint32_t        _pad;
    const uint32_t *accum;           /* host ptr [n_accum], each ≥ 1            */
    const uint64_t *shard_bytes;     /* host ptr [nM][8] (row m: S_d of Ms[m]'s
                                        placement, d < Ms[m]) or NULL ⇒ every
                                        device all-reduces grad_bytes       */
} pp_scenario;

typedef struct {
    uint64_t C_lo, C_hi;             /* C as u128 (ps × µ-epochs)               */
    uint64_t step_ps, steps, uepochs;
    uint32_t feasible, accum;        /* accum: the chosen a (0 if infeasible)   */
} pp_cell;

/* S_d = Σ param_bytes of the ops placed on device d (R24).  placement: host
 * ptr uint8 [K] descriptor order, values < M; out: host ptr uint64 [8].     */
int pp_shard_bytes(const pp_dfg *dfg, int M, const uint8_t *placement, uint64_t *out);

/* Ms, T_M_ps: host ptrs [nM] (nM ∈ [1,8], each M ≥ 1, T_M > 0);
 * d_cells: device ptr pp_cell [nM][N_max], cell (m, N) at m·N_max + N−1;
 * N_max ∈ [1, 65536].  Synchronises cuda_stream (to report PP_E_RANGE).     */
int pp_project_e2e(const pp_scenario *sc, int nM, const uint32_t *Ms, const uint64_t *T_M_ps,
                   uint32_t N_max, pp_cell *d_cells, void *cuda_stream);

/* Crossover (Eq. 6, strict; §5; R16):
 *   n_star_M[m]   = min{N : C(M_m,N) < C(1,N), both feasible}, 0 = none
 *   persistent_M  = 1 iff the hybrid stays strictly better at every N ≥ n_star_M
 *   n_star        = min over M ≥ 2; m_at_n_star = the M with least C there
 *                   (ties → smaller M)
 *   n_star_vs_best_dp = min{N : min_M C(M,N) < min_{N'≤N} C(1,N')}
 * Ms must contain 1.  d_best_m: optional device ptr uint32 [N_max] (M with the
 * least C at each N, ties → smaller M, 0 = no feasible cell).  *out is a
 * host ptr.  Synchronises cuda_stream.                                       */
typedef struct {
    uint32_t n_star, m_at_n_star;
    uint32_t n_star_M[8], persistent_M[8];
    uint32_t n_star_vs_best_dp;
} pp_crossover_result;

int pp_crossover(const pp_cell *d_cells, int nM, const uint32_t *Ms, uint32_t N_max,
                 pp_crossover_result *out, uint32_t *d_best_m, void *cuda_stream);

/* Message of the last failing call on this thread ("" if none). */
const char *pp_last_error(void);

/* Number of kernel launches issued by this library since load (for the
 * benchmark's gpu_launches count). */
uint64_t pp_kernel_launch_count(void);

/* Optional timing of the search kernel inside pp_search_best: when enabled,
 * a CUDA event pair brackets every search-kernel launch on the caller's
 * stream and the elapsed times are accumulated (read after the call, which
 * synchronises).  Enabling resets the accumulators.  Not thread-safe.     */
void pp_set_kernel_timing(int enable);
void pp_get_kernel_timing(double *total_ms, uint64_t *timed_launches);

#ifdef __cplusplus
}
#endif
#endif /* PP_H */
