/*
 * pp_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of what the hot path of
 * arXiv 1907.13257 computes (as read in SURVEY.md §8(c), readings R1–R20,
 * definitions O1–O12).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant generator with the CUDA path in
 * paper_1907_13257_b200/ and neither side imports the other.
 *
 * Arithmetic: unsigned 64-bit integers for times (picoseconds), unsigned
 * __int128 for products.  No floating point anywhere in a compared result.
 *
 * Citations: "PAPER.md:L" are line numbers of /root/reference/PAPER.md with
 * the section/equation they fall in; "SPEC.md:L" likewise for SPEC.md.
 *
 * Parity status per function (see DESIGN.md §Oracle pins):
 *   or_prepare / or_pi         pinned (SPEC Kahn examples, brute-force tests)
 *   or_schedule                pinned (K1–K7, brute-force longest path, invariants)
 *   or_gen (GRAY)              pinned (Gray property: one digit changes per step,
 *                              bijection onto [0,M)^K; M=2 equals i^(i>>1))
 *   or_gen (RANDOM, PERTURB)   pinned (seeds chosen so the generator word IS a
 *                              published SplitMix64 output: the expected bits /
 *                              bytes of the placement come from that literal;
 *                              distribution and flip-rate properties)
 *   or_round / or_search       pinned (K2, K3, K8, exhaustive == brute force)
 *   or_ar                      pinned (K9 closed form)
 *   or_epochs / or_cell        pinned (K10–K12 paper ratios)
 *   or_crossover               pinned (K10–K14 paper statements)
 *   or_prepare_hw              pinned (SPEC route examples, closed forms on
 *                              ring/switch/two-node graphs, Floyd–Warshall)
 *   or_eft                     pinned (SPEC heuristic_place examples, closed
 *                              forms: round-robin of equal independent ops,
 *                              chain kept whole, diamond → (0,0,1,1))
 *   or_pipeline(_search)       pinned (GPipe bubble closed form, M = 1,
 *                              discrete-event simulation, exhaustive brute)
 *   or_exact / or_round_exact  pinned (SPEC exact_schedule examples, a hand
 *                              case where in-order issue loses, brute force
 *                              over per-device orders, exact ≤ in-order)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

typedef unsigned __int128 u128;

#define OR_OK 0
#define OR_E_INVALID (-1)
#define OR_E_CYCLE (-2)
#define OR_E_RANGE (-3)
#define OR_E_TOO_LARGE (-4)
#define OR_E_INFEASIBLE (-5)

#define OR_INFEASIBLE_MAKESPAN UINT64_MAX

/* ---------------------------------------------------------------- O1 inputs */
/* PAPER.md:350 (§6): DFG vertices K with Δ(k) and M(k), edges E with D(e);
 * links with bandwidth B(l); Table 2 PAPER.md:365–392.
 * R1: every op has a forward time Δf and a backward time Δb; every edge has
 * activation bytes D_f and gradient bytes D_b (default D_b = D_f).           */
typedef struct {
    int32_t K, E;
    const int64_t *op_id;          /* external ids, NULL => 0..K-1 */
    const uint64_t *fwd_ps;        /* Δf(k) */
    const uint64_t *bwd_ps;        /* Δb(k) */
    const uint64_t *mem_bytes;     /* M(k), NULL => 0 */
    const uint64_t *param_bytes;   /* weight bytes, NULL => 0 */
    const int32_t *edge_src, *edge_dst;
    const uint64_t *edge_fwd_bytes;
    const uint64_t *edge_bwd_bytes; /* NULL => = fwd */
    uint64_t link_bw_Bps, link_lat_ps, dev_mem_cap_bytes; /* cap 0 = unlimited */
} or_input;

typedef struct {
    int K, E;
    int64_t *id;        /* external id, original index order */
    int *pi;            /* pi[p]  = original index of the op at π position p */
    int *pos;           /* pos[k] = π position of original op k            */
    /* everything below is indexed by π position */
    uint64_t *df, *db, *mem, *param;
    /* adjacency lists by π position: in-edges and out-edges */
    int *in_cnt, **in_src;  uint64_t **in_cf;
    int *out_cnt, **out_dst; uint64_t **out_cb;
    uint64_t cap;
    uint64_t t1;
    uint64_t grad_bytes;
    /* general hardware graph (NEXT f2): per-edge cost for every ordered
     * device pair, cfm[(eid·nd + a)·nd + b]; adjacency lists carry edge ids */
    int nd;                 /* 0 = one uniform hop (R4) */
    /* pipeline MP (NEXT f3): edges by π position, bytes, the uniform link */
    int *e_src, *e_dst;
    uint64_t *e_bf, *e_bb;
    uint64_t link_bw, link_lat;
    int **in_eid, **out_eid;
    uint64_t *cfm, *cbm;
} or_ctx;

/* Hardware graph of PAPER.md:352 (§6): devices 0..nd−1, routers nd..nd+R−1,
 * bidirectional links with bandwidth B(l) > 0 and latency L(l).             */
typedef struct {
    int32_t num_devices, num_routers, num_links;
    const int32_t *link_a, *link_b;
    const uint64_t *link_bw_Bps, *link_lat_ps;
    uint64_t dev_mem_cap_bytes;
} or_hw;

typedef struct { uint64_t makespan, index; } or_best;   /* an argmin (O7) */

static void set_err(char *err, int errlen, const char *msg) {
    if (err && errlen > 0) { strncpy(err, msg, (size_t)errlen - 1); err[errlen - 1] = 0; }
}

/* O3: c(e) = ⌈D(e)·10^12 / BW⌉ + L  (§6 Δ_e = Σ_l C_el·(D(e)/B(l)+L(l)),
 * reduced to one logical hop by reading R4).                                  */
uint64_t or_edge_cost(uint64_t bytes, uint64_t bw, uint64_t lat, int *overflow) {
    u128 num = (u128)bytes * (u128)1000000000000ULL;
    u128 q = num / bw;
    if (num % bw) q += 1;
    q += lat;
    if (q >> 64) { if (overflow) *overflow = 1; return UINT64_MAX; }
    return (uint64_t)q;
}

void or_free(or_ctx *c) {
    if (!c) return;
    for (int p = 0; p < c->K; p++) {
        if (c->in_src) free(c->in_src[p]);
        if (c->in_cf) free(c->in_cf[p]);
        if (c->out_dst) free(c->out_dst[p]);
        if (c->out_cb) free(c->out_cb[p]);
    }
    if (c->in_eid) for (int p = 0; p < c->K; p++) { free(c->in_eid[p]); free(c->out_eid[p]); }
    free(c->in_eid); free(c->out_eid); free(c->cfm); free(c->cbm);
    free(c->in_src); free(c->in_cf); free(c->out_dst); free(c->out_cb);
    free(c->e_src); free(c->e_dst); free(c->e_bf); free(c->e_bb);
    free(c->in_cnt); free(c->out_cnt);
    free(c->id); free(c->pi); free(c->pos); free(c->df); free(c->db); free(c->mem); free(c->param);
    free(c);
}

/* O2: π = Kahn's algorithm; among ready ops pop the smallest external id
 * (reading R3).  Plain O(K^2) selection.                      */
static int kahn(int K, int E, const int64_t *id, const int32_t *src, const int32_t *dst,
                int *pi, char *err, int errlen) {
    int *indeg = calloc((size_t)K, sizeof(int));
    char *done = calloc((size_t)K, 1);
    for (int e = 0; e < E; e++) indeg[dst[e]]++;
    int n = 0;
    while (n < K) {
        int best = -1;
        for (int k = 0; k < K; k++)
            if (!done[k] && indeg[k] == 0 && (best < 0 || id[k] < id[best])) best = k;
        if (best < 0) break;
        done[best] = 1;
        pi[n++] = best;
        for (int e = 0; e < E; e++) if (src[e] == best) indeg[dst[e]]--;
    }
    if (n < K) {
        /* report one cycle: walk backwards along unfinished
         * predecessors from any unfinished op until an op repeats            */
        int *seen = malloc(sizeof(int) * (size_t)K);
        for (int k = 0; k < K; k++) seen[k] = -1;
        int v = -1;
        for (int k = 0; k < K; k++) if (!done[k]) { v = k; break; }
        int step = 0;
        while (seen[v] < 0) {
            seen[v] = step++;
            int u = -1;
            for (int e = 0; e < E; e++) if (dst[e] == v && !done[src[e]]) { u = src[e]; break; }
            v = u;
        }
        /* v is on the cycle: collect it */
        char msg[512]; int off = snprintf(msg, sizeof msg, "cycle:");
        int start = v, guard = 0;
        do {
            off += snprintf(msg + off, sizeof msg - (size_t)off, " %lld", (long long)id[v]);
            int u = -1;
            for (int e = 0; e < E; e++) if (dst[e] == v && !done[src[e]]) { u = src[e]; break; }
            v = u; guard++;
        } while (v != start && guard <= K && off < 480);
        set_err(err, errlen, msg);
        free(seen); free(indeg); free(done);
        return OR_E_CYCLE;
    }
    free(indeg); free(done);
    return OR_OK;
}

int or_prepare(const or_input *in, or_ctx **out, char *err, int errlen) {
    *out = NULL;
    int K = in->K, E = in->E;
    if (K < 1 || E < 0 || !in->fwd_ps || !in->bwd_ps || (E > 0 && (!in->edge_src || !in->edge_dst || !in->edge_fwd_bytes))) {
        set_err(err, errlen, "invalid sizes or null arrays"); return OR_E_INVALID;
    }
    if (in->link_bw_Bps == 0) { set_err(err, errlen, "link bandwidth must be > 0"); return OR_E_INVALID; }
    int64_t *id = malloc(sizeof(int64_t) * (size_t)K);
    for (int k = 0; k < K; k++) id[k] = in->op_id ? in->op_id[k] : k;
    for (int k = 0; k < K; k++) {
        if (id[k] < 0) { set_err(err, errlen, "negative op id"); free(id); return OR_E_INVALID; }
        for (int j = 0; j < k; j++)
            if (id[j] == id[k]) { set_err(err, errlen, "duplicate op id"); free(id); return OR_E_INVALID; }
    }
    for (int e = 0; e < E; e++) {
        if (in->edge_src[e] < 0 || in->edge_src[e] >= K || in->edge_dst[e] < 0 || in->edge_dst[e] >= K) {
            set_err(err, errlen, "dangling edge endpoint"); free(id); return OR_E_INVALID;
        }
        if (in->edge_src[e] == in->edge_dst[e]) { set_err(err, errlen, "self edge"); free(id); return OR_E_INVALID; }
    }
    int *pi = malloc(sizeof(int) * (size_t)K);
    int rc = kahn(K, E, id, in->edge_src, in->edge_dst, pi, err, errlen);
    if (rc) { free(id); free(pi); return rc; }

    or_ctx *c = calloc(1, sizeof(or_ctx));
    c->K = K; c->E = E; c->id = id; c->pi = pi;
    c->pos = malloc(sizeof(int) * (size_t)K);
    for (int p = 0; p < K; p++) c->pos[pi[p]] = p;
    c->df = malloc(8 * (size_t)K); c->db = malloc(8 * (size_t)K); c->mem = malloc(8 * (size_t)K);
    c->param = malloc(8 * (size_t)K);
    for (int p = 0; p < K; p++) {
        int k = pi[p];
        c->df[p] = in->fwd_ps[k];
        c->db[p] = in->bwd_ps[k];
        c->mem[p] = in->mem_bytes ? in->mem_bytes[k] : 0;
        c->param[p] = in->param_bytes ? in->param_bytes[k] : 0;
    }
    c->cap = in->dev_mem_cap_bytes;
    c->in_cnt = calloc((size_t)K, sizeof(int)); c->out_cnt = calloc((size_t)K, sizeof(int));
    c->in_src = calloc((size_t)K, sizeof(int *)); c->in_cf = calloc((size_t)K, sizeof(uint64_t *));
    c->out_dst = calloc((size_t)K, sizeof(int *)); c->out_cb = calloc((size_t)K, sizeof(uint64_t *));
    for (int e = 0; e < E; e++) { c->in_cnt[c->pos[in->edge_dst[e]]]++; c->out_cnt[c->pos[in->edge_src[e]]]++; }
    for (int p = 0; p < K; p++) {
        c->in_src[p] = malloc(sizeof(int) * (size_t)(c->in_cnt[p] + 1));
        c->in_cf[p] = malloc(8 * (size_t)(c->in_cnt[p] + 1));
        c->out_dst[p] = malloc(sizeof(int) * (size_t)(c->out_cnt[p] + 1));
        c->out_cb[p] = malloc(8 * (size_t)(c->out_cnt[p] + 1));
        c->in_cnt[p] = 0; c->out_cnt[p] = 0;
    }
    /* O3 edge costs, and the R3/range bound: Σ(Δf+Δb) + Σ(c_f+c_b) < 2^61 */
    u128 bound = 0;
    int ovf = 0;
    c->e_src = malloc(sizeof(int) * (size_t)(E + 1)); c->e_dst = malloc(sizeof(int) * (size_t)(E + 1));
    c->e_bf = malloc(8 * (size_t)(E + 1)); c->e_bb = malloc(8 * (size_t)(E + 1));
    c->link_bw = in->link_bw_Bps; c->link_lat = in->link_lat_ps;
    for (int e = 0; e < E; e++) {
        int u = c->pos[in->edge_src[e]], v = c->pos[in->edge_dst[e]];
        uint64_t bf = in->edge_fwd_bytes[e];
        uint64_t bb = in->edge_bwd_bytes ? in->edge_bwd_bytes[e] : bf;
        c->e_src[e] = u; c->e_dst[e] = v; c->e_bf[e] = bf; c->e_bb[e] = bb;
        uint64_t cf = or_edge_cost(bf, in->link_bw_Bps, in->link_lat_ps, &ovf);
        uint64_t cb = or_edge_cost(bb, in->link_bw_Bps, in->link_lat_ps, &ovf);
        c->in_src[v][c->in_cnt[v]] = u; c->in_cf[v][c->in_cnt[v]] = cf; c->in_cnt[v]++;
        c->out_dst[u][c->out_cnt[u]] = v; c->out_cb[u][c->out_cnt[u]] = cb; c->out_cnt[u]++;
        bound += (u128)cf + cb;
    }
    u128 t1 = 0;
    for (int p = 0; p < K; p++) t1 += (u128)c->df[p] + c->db[p];
    bound += t1;
    if (ovf || (bound >> 61)) { set_err(err, errlen, "time bound >= 2^61 ps"); or_free(c); return OR_E_RANGE; }
    c->t1 = (uint64_t)t1;
    c->grad_bytes = 0;
    if (in->param_bytes) for (int k = 0; k < K; k++) c->grad_bytes += in->param_bytes[k];
    *out = c;
    return OR_OK;
}

/* NEXT f2 — the general hardware graph (Δ_e = Σ_l C_el·(D(e)/B(l)
 * + L(l))).  Reading: a transfer uses the delay-shortest
 * route for its payload (with no link contention, R5, this is
 * what the ILP optimum picks), each hop charged ⌈D·10^12/B(l)⌉ + L(l) ps:
 *   c(e, a, b) = min over paths a → b of Σ_hops (⌈D(e)·10^12/B⌉ + L).
 * Plain Dijkstra (O(V^2)) per edge, per direction and per source device.     */
static u128 dijkstra_cost(const or_hw *hw, uint64_t bytes, int src, int dst) {
    int V = hw->num_devices + hw->num_routers;
    u128 *dist = malloc(sizeof(u128) * (size_t)V);
    char *done = calloc((size_t)V, 1);
    const u128 INF = ~(u128)0;
    for (int v = 0; v < V; v++) dist[v] = INF;
    dist[src] = 0;
    for (int it = 0; it < V; it++) {
        int u = -1;
        for (int v = 0; v < V; v++) if (!done[v] && dist[v] != INF && (u < 0 || dist[v] < dist[u])) u = v;
        if (u < 0) break;
        done[u] = 1;
        for (int l = 0; l < hw->num_links; l++) {
            int a = hw->link_a[l], b = hw->link_b[l], v;
            if (a == u) v = b; else if (b == u) v = a; else continue;
            u128 w = ((u128)bytes * 1000000000000ULL + hw->link_bw_Bps[l] - 1) / hw->link_bw_Bps[l] + hw->link_lat_ps[l];
            if (dist[u] + w < dist[v]) dist[v] = dist[u] + w;
        }
    }
    u128 r = dist[dst];
    free(dist); free(done);
    return r;
}

int or_prepare_hw(const or_input *in, const or_hw *hw, or_ctx **out, char *err, int errlen) {
    *out = NULL;
    if (!hw || hw->num_devices < 1 || hw->num_devices > 8 || hw->num_routers < 0 || hw->num_links < 0) {
        set_err(err, errlen, "invalid hardware graph sizes"); return OR_E_INVALID;
    }
    int V = hw->num_devices + hw->num_routers;
    for (int l = 0; l < hw->num_links; l++) {
        if (hw->link_a[l] < 0 || hw->link_a[l] >= V || hw->link_b[l] < 0 || hw->link_b[l] >= V ||
            hw->link_a[l] == hw->link_b[l] || hw->link_bw_Bps[l] == 0) {
            set_err(err, errlen, "invalid link"); return OR_E_INVALID;
        }
    }
    /* the DFG part, with a dummy uniform link (costs replaced below) */
    or_input in2 = *in;
    in2.link_bw_Bps = 1000000000000ULL;
    in2.link_lat_ps = 0;
    in2.dev_mem_cap_bytes = hw->dev_mem_cap_bytes;
    int rc = or_prepare(&in2, out, err, errlen);
    if (rc) return rc;
    or_ctx *c = *out;
    int nd = hw->num_devices, E = c->E, K = c->K;
    for (int a = 0; a < nd; a++)
        for (int b = 0; b < nd; b++)
            if (a != b && dijkstra_cost(hw, 0, a, b) == ~(u128)0) {
                set_err(err, errlen, "devices not connected"); or_free(c); *out = NULL; return OR_E_INVALID;
            }
    c->nd = nd;
    c->cfm = calloc((size_t)E * nd * nd + 1, 8);
    c->cbm = calloc((size_t)E * nd * nd + 1, 8);
    u128 bound = c->t1;
    for (int e = 0; e < E; e++) {
        uint64_t bf = in->edge_fwd_bytes[e], bb = in->edge_bwd_bytes ? in->edge_bwd_bytes[e] : bf;
        u128 mf = 0, mb = 0;
        for (int a = 0; a < nd; a++)
            for (int b = 0; b < nd; b++) {
                if (a == b) continue;
                u128 f = dijkstra_cost(hw, bf, a, b), g = dijkstra_cost(hw, bb, a, b);
                if ((f >> 64) || (g >> 64)) { set_err(err, errlen, "edge cost overflow"); or_free(c); *out = NULL; return OR_E_RANGE; }
                c->cfm[((size_t)e * nd + a) * nd + b] = (uint64_t)f;
                c->cbm[((size_t)e * nd + a) * nd + b] = (uint64_t)g;
                if (f > mf) mf = f;
                if (g > mb) mb = g;
            }
        bound += mf + mb;
    }
    if (bound >> 61) { set_err(err, errlen, "time bound >= 2^61 ps"); or_free(c); *out = NULL; return OR_E_RANGE; }
    /* adjacency lists with edge ids, in the same order as in_src / out_dst */
    c->in_eid = calloc((size_t)K, sizeof(int *));
    c->out_eid = calloc((size_t)K, sizeof(int *));
    int *ic = calloc((size_t)K, sizeof(int)), *oc = calloc((size_t)K, sizeof(int));
    for (int p = 0; p < K; p++) {
        c->in_eid[p] = malloc(sizeof(int) * (size_t)(c->in_cnt[p] + 1));
        c->out_eid[p] = malloc(sizeof(int) * (size_t)(c->out_cnt[p] + 1));
    }
    for (int e = 0; e < E; e++) {
        int u = c->pos[in->edge_src[e]], v = c->pos[in->edge_dst[e]];
        c->in_eid[v][ic[v]++] = e;
        c->out_eid[u][oc[u]++] = e;
    }
    free(ic); free(oc);
    return OR_OK;
}

uint64_t or_hw_edge_cost(const or_ctx *c, int e, int a, int b, int bwd) {
    if (!c->nd || a == b) return 0;
    return (bwd ? c->cbm : c->cfm)[((size_t)e * c->nd + a) * c->nd + b];
}

int or_num_ops(const or_ctx *c) { return c->K; }
void or_get_pi(const or_ctx *c, int32_t *pi_out) { for (int p = 0; p < c->K; p++) pi_out[p] = c->pi[p]; }
/* O4 / R8: T_1 = Σ_k (Δf(k)+Δb(k)), the all-on-one-device makespan (PAPER.md:501 assumption 1). */
uint64_t or_t1(const or_ctx *c) { return c->t1; }
uint64_t or_grad_bytes(const or_ctx *c) { return c->grad_bytes; }

/* O4: the in-order list schedule of placement d (indexed by π position).
 * Forward in π order, backward in reverse π order (R1, R2):
 *   PAPER.md:443–453 dependency T(dst) ≥ T(src)+Δ(src)+Δ_e,
 *   PAPER.md:465–476 one op at a time per device,
 *   PAPER.md:497–503 back-to-back ops; comm overlaps compute.
 * start_f / start_b (optional) receive each op's start times.               */
uint64_t or_schedule_ex(const or_ctx *c, int M, const uint8_t *d,
                        uint64_t *start_f, uint64_t *start_b) {
    int K = c->K;
    uint64_t *fin = calloc((size_t)K, 8), *finb = calloc((size_t)K, 8);
    uint64_t free_t[256];
    for (int m = 0; m < M; m++) free_t[m] = 0;
    for (int p = 0; p < K; p++) {                       /* forward */
        uint64_t r = 0;
        for (int i = 0; i < c->in_cnt[p]; i++) {
            int u = c->in_src[p][i];
            uint64_t cost = c->nd ? c->cfm[((size_t)c->in_eid[p][i] * c->nd + d[u]) * c->nd + d[p]] : c->in_cf[p][i];
            uint64_t t = fin[u] + (d[u] != d[p] ? cost : 0);
            if (t > r) r = t;
        }
        uint64_t s = r > free_t[d[p]] ? r : free_t[d[p]];
        if (start_f) start_f[p] = s;
        fin[p] = s + c->df[p];
        free_t[d[p]] = fin[p];
    }
    for (int p = K - 1; p >= 0; p--) {                  /* backward */
        uint64_t r = (c->out_cnt[p] == 0) ? fin[p] : 0;  /* a sink waits for its own forward (R1) */
        for (int i = 0; i < c->out_cnt[p]; i++) {
            int w = c->out_dst[p][i];
            uint64_t cost = c->nd ? c->cbm[((size_t)c->out_eid[p][i] * c->nd + d[w]) * c->nd + d[p]] : c->out_cb[p][i];
            uint64_t t = finb[w] + (d[w] != d[p] ? cost : 0);
            if (t > r) r = t;
        }
        uint64_t s = r > free_t[d[p]] ? r : free_t[d[p]];
        if (start_b) start_b[p] = s;
        finb[p] = s + c->db[p];
        free_t[d[p]] = finb[p];
    }
    uint64_t mk = 0;
    for (int m = 0; m < M; m++) if (free_t[m] > mk) mk = free_t[m];
    free(fin); free(finb);
    /* PAPER.md:478–487 memory capacity, reading R7: violation => infeasible */
    if (c->cap > 0) {
        for (int m = 0; m < M; m++) {
            u128 used = 0;
            for (int p = 0; p < K; p++) if (d[p] == m) used += c->mem[p];
            if (used > c->cap) return OR_INFEASIBLE_MAKESPAN;
        }
    }
    return mk;
}

uint64_t or_schedule(const or_ctx *c, int M, const uint8_t *d_pi) {
    return or_schedule_ex(c, M, d_pi, NULL, NULL);
}

/* placement given in original (descriptor) op order */
int or_makespan_orig(const or_ctx *c, int M, const uint8_t *d_orig, uint64_t *out) {
    if (M < 1 || M > 8 || (c->nd && M > c->nd)) return OR_E_INVALID;
    uint8_t *d = malloc((size_t)c->K);
    for (int p = 0; p < c->K; p++) {
        d[p] = d_orig[c->pi[p]];
        if (d[p] >= M) { free(d); return OR_E_INVALID; }
    }
    *out = or_schedule(c, M, d);
    free(d);
    return OR_OK;
}

/* ------------------------------------------- NEXT f1: the exact schedule */
/* The makespan-optimal schedule of a FIXED placement: DLPlacer "minimizes
 * per step training time by ... determining the execution start time of each
 * vertex on a device" (§6) subject to the dependency constraint
 * (PAPER.md:443–453), the non-overlap constraint and the
 * back-to-back assumption; SPEC.md:161–169 exact_schedule.
 *
 * Nodes: F_p (forward of π position p) and B_p (its backward), on device d[p].
 * Arcs (R1): F_u → F_v with c_f(e) when cut, B_v → B_u with c_b(e) when cut,
 * F_p → B_p.  Reading R22: a schedule is a linear extension σ of the arcs;
 * each node starts at max(data ready, finish of the node before it on its
 * device in σ).  Every feasible schedule's per-device orders are induced by
 * some σ, whose schedule is no later, so the optimum is
 *     exact = min over all linear extensions σ of makespan(σ).
 * Enumerated by depth-first search over σ.  A branch stops when it cannot
 * beat the best complete σ: (a) its partial makespan (max finish so far) is
 * already ≥ best — extending σ never lowers a finish time already fixed; or
 * (b) some device's free time plus the work still to run on it is ≥ best —
 * every remaining node of that device starts after its free time and they
 * run one at a time.  Exponential: small DFGs only.      */
typedef struct {
    const or_ctx *c;
    const uint8_t *d;
    int K;
    uint64_t *fin;        /* [2K] finish time of each scheduled node            */
    uint8_t *done;        /* [2K]                                              */
    uint64_t free_t[8];
    uint64_t left[8];     /* work not yet scheduled, per device */
    int M;
    uint64_t best;
} or_ex;

/* data-ready time of node n if all its predecessors are done; 0 with *ok=0 otherwise */
static uint64_t ex_ready(const or_ex *x, int n, int *ok) {
    const or_ctx *c = x->c;
    const uint8_t *d = x->d;
    int K = x->K;
    uint64_t r = 0;
    *ok = 1;
    if (n < K) {                                   /* F_p: forward in-edges */
        int p = n;
        for (int i = 0; i < c->in_cnt[p]; i++) {
            int u = c->in_src[p][i];
            if (!x->done[u]) { *ok = 0; return 0; }
            uint64_t cost = c->nd ? c->cfm[((size_t)c->in_eid[p][i] * c->nd + d[u]) * c->nd + d[p]] : c->in_cf[p][i];
            uint64_t t = x->fin[u] + (d[u] != d[p] ? cost : 0);
            if (t > r) r = t;
        }
    } else {                                       /* B_p: own forward + gradients */
        int p = n - K;
        if (!x->done[p]) { *ok = 0; return 0; }
        r = x->fin[p];
        for (int i = 0; i < c->out_cnt[p]; i++) {
            int w = c->out_dst[p][i];
            if (!x->done[K + w]) { *ok = 0; return 0; }
            uint64_t cost = c->nd ? c->cbm[((size_t)c->out_eid[p][i] * c->nd + d[w]) * c->nd + d[p]] : c->out_cb[p][i];
            uint64_t t = x->fin[K + w] + (d[w] != d[p] ? cost : 0);
            if (t > r) r = t;
        }
    }
    return r;
}

static void ex_dfs(or_ex *x, int placed, uint64_t partial) {
    int K = x->K;
    if (placed == 2 * K) {
        if (partial < x->best) x->best = partial;
        return;
    }
    for (int n = 0; n < 2 * K; n++) {
        if (x->done[n]) continue;
        int ok;
        uint64_t r = ex_ready(x, n, &ok);
        if (!ok) continue;
        int p = n < K ? n : n - K;
        int dev = x->d[p];
        uint64_t s = r > x->free_t[dev] ? r : x->free_t[dev];
        uint64_t f = s + (n < K ? x->c->df[p] : x->c->db[p]);
        uint64_t np = f > partial ? f : partial;
        if (np >= x->best) continue;               /* (a) */
        uint64_t dur = n < K ? x->c->df[p] : x->c->db[p];
        uint64_t saved = x->free_t[dev];
        x->fin[n] = f;
        x->done[n] = 1;
        x->free_t[dev] = f;
        x->left[dev] -= dur;
        int hopeless = 0;                          /* (b) */
        for (int m = 0; m < x->M; m++)
            if (x->free_t[m] + x->left[m] >= x->best) hopeless = 1;
        if (!hopeless) ex_dfs(x, placed + 1, np);
        x->left[dev] += dur;
        x->free_t[dev] = saved;
        x->done[n] = 0;
    }
}

/* exact makespan of placement d (by π position); OR_INFEASIBLE_MAKESPAN when
 * the memory cap is violated (R7)                          */
uint64_t or_exact(const or_ctx *c, int M, const uint8_t *d) {
    int K = c->K;
    if (c->cap > 0) {
        for (int m = 0; m < M; m++) {
            u128 used = 0;
            for (int p = 0; p < K; p++) if (d[p] == m) used += c->mem[p];
            if (used > c->cap) return OR_INFEASIBLE_MAKESPAN;
        }
    }
    or_ex x;
    memset(&x, 0, sizeof x);
    x.c = c; x.d = d; x.K = K; x.M = M;
    for (int p = 0; p < K; p++) x.left[d[p]] += c->df[p] + c->db[p];
    x.fin = calloc((size_t)(2 * K) + 1, 8);
    x.done = calloc((size_t)(2 * K) + 1, 1);
    x.best = UINT64_MAX;
    ex_dfs(&x, 0, 0);
    free(x.fin); free(x.done);
    return x.best;
}

int or_makespan_exact_orig(const or_ctx *c, int M, const uint8_t *d_orig, uint64_t *out) {
    if (M < 1 || M > 8 || (c->nd && M > c->nd)) return OR_E_INVALID;
    uint8_t *d = malloc((size_t)c->K + 1);
    for (int p = 0; p < c->K; p++) {
        d[p] = d_orig[c->pi[p]];
        if (d[p] >= M) { free(d); return OR_E_INVALID; }
    }
    *out = or_exact(c, M, d);
    free(d);
    return OR_OK;
}

/* ----------------------------------------- NEXT f4: EFT-greedy base seed */
/* SPEC.md:245–253 heuristic_place: "earliest-finish-time greedy in
 * topological order: each vertex assigned to the device minimizing its
 * completion time given current partial schedule and incoming-edge
 * communication delays; memory-feasible".  Reading R23: the forward pass in
 * π order decides (the backward ops follow their forward op's device);
 * ties go to the smallest device; a device whose memory would exceed the cap
 * is skipped; no feasible device => OR_E_INFEASIBLE.
 * d_out receives the placement by π position.                                */
int or_eft(const or_ctx *c, int M, uint8_t *d_out) {
    int K = c->K;
    if (M < 1 || M > 8 || (c->nd && M > c->nd)) return OR_E_INVALID;
    uint64_t *fin = calloc((size_t)K + 1, 8);
    uint64_t free_t[8] = {0};
    u128 used[8] = {0};
    for (int p = 0; p < K; p++) {
        int best_m = -1;
        uint64_t best_f = 0;
        for (int m = 0; m < M; m++) {
            if (c->cap > 0 && used[m] + c->mem[p] > c->cap) continue;
            uint64_t r = 0;
            for (int i = 0; i < c->in_cnt[p]; i++) {
                int u = c->in_src[p][i];
                uint64_t cost = c->nd ? c->cfm[((size_t)c->in_eid[p][i] * c->nd + d_out[u]) * c->nd + m]
                                      : c->in_cf[p][i];
                uint64_t t = fin[u] + (d_out[u] != m ? cost : 0);
                if (t > r) r = t;
            }
            uint64_t st = r > free_t[m] ? r : free_t[m];
            uint64_t f = st + c->df[p];
            if (best_m < 0 || f < best_f) { best_m = m; best_f = f; }
        }
        if (best_m < 0) { free(fin); return OR_E_INFEASIBLE; }
        d_out[p] = (uint8_t)best_m;
        fin[p] = best_f;
        free_t[best_m] = best_f;
        used[best_m] += c->mem[p];
    }
    free(fin);
    return OR_OK;
}

int or_eft_orig(const or_ctx *c, int M, uint8_t *d_orig) {
    uint8_t *d = malloc((size_t)c->K + 1);
    int rc = or_eft(c, M, d);
    if (rc == OR_OK) for (int p = 0; p < c->K; p++) d_orig[c->pi[p]] = d[p];
    free(d);
    return rc;
}

/* NEXT f4 (reading R24): gradient shard of each device under a placement,
 * S_d = Σ param_bytes of the ops on device d (descriptor order placement).   */
int or_shard_bytes(const or_ctx *c, int M, const uint8_t *d_orig, uint64_t *out8) {
    if (M < 1 || M > 8) return OR_E_INVALID;
    for (int m = 0; m < 8; m++) out8[m] = 0;
    for (int p = 0; p < c->K; p++) {
        int k = c->pi[p];
        if (d_orig[k] >= M) return OR_E_INVALID;
        out8[d_orig[k]] += c->param[p];
    }
    return OR_OK;
}

/* ------------------------------------------ NEXT f3: pipeline-parallel MP */
/* GPipe-style pipelining (§2: "Networks are partitioned into
 * groups containing one or a few layers of the network, where each group is
 * placed on a different device ... a mini-batch is split into yet smaller
 * micro-batches and each device processes a different micro-batch
 * sequentially but concurrently"; §4.4: GNMT and BigLSTM are
 * split by pipelining).  Reading R26:
 *   stage s = π positions [cut_s, cut_{s+1}), cut_0 = 0 < cut_1 < … < cut_M = K,
 *     on device s (π is topological, so every edge goes to the same or a
 *     later stage);
 *   per micro-batch: tf_s = ⌈Σ_{p∈s} Δf(p) / m⌉ + n_s·o, tb_s = ⌈Σ Δb / m⌉ + n_s·o
 *     (n_s ops in the stage; o = a fixed per-op cost each micro-batch pays,
 *     the "kernel overheads" of PAPER.md:299, reading R27; o = 0 by default);
 *   a → b (a < b) carries the micro-batch's activations of every edge from a
 *     to b as one transfer of ⌈D_ab·10^12 / (m·BW)⌉ + L ps (D_ab = Σ D_f), the
 *     gradients back from b to a likewise with Σ D_b; no edge, no transfer;
 *   forward, micro-batches j = 0..m−1 in order:
 *     F[s][j] = max(F[s][j−1], max_{a<s} F[a][j] + cf(a,s)) + tf_s
 *   backward after the forward flush, micro-batches in reverse order:
 *     B[s][j] = max(B[s][j+1], max_{b>s} B[b][j] + cb(b,s)) + tb_s,
 *     B[s][m] := F[s][m−1]   (each device runs its ops one at a time)
 *   makespan = max_s B[s][0]; a stage whose Σ M(k) exceeds the cap makes the
 *   pipeline infeasible.                                 */
uint64_t or_pipeline_ex(const or_ctx *c, int M, const int32_t *cuts, uint32_t m, uint64_t o) {
    int K = c->K;
    if (M < 1 || M > 8 || M > K || m < 1 || m > 65536 || c->nd) return OR_INFEASIBLE_MAKESPAN;  /* invalid */
    for (int s = 0; s < M - 1; s++)
        if (cuts[s] < 1 || cuts[s] > K - 1 || (s > 0 && cuts[s] <= cuts[s - 1])) return OR_INFEASIBLE_MAKESPAN;
    int st[9];
    st[0] = 0; st[M] = K;
    for (int s = 1; s < M; s++) st[s] = cuts[s - 1];
    int *stage_of = malloc(sizeof(int) * (size_t)K);
    for (int s = 0; s < M; s++) for (int p = st[s]; p < st[s + 1]; p++) stage_of[p] = s;
    uint64_t tf[8], tb[8];
    for (int s = 0; s < M; s++) {
        u128 sf = 0, sb = 0, mem = 0;
        for (int p = st[s]; p < st[s + 1]; p++) { sf += c->df[p]; sb += c->db[p]; mem += c->mem[p]; }
        if (c->cap > 0 && mem > c->cap) { free(stage_of); return OR_INFEASIBLE_MAKESPAN; }
        uint64_t n_s = (uint64_t)(st[s + 1] - st[s]);
        tf[s] = (uint64_t)((sf + m - 1) / m) + n_s * o;
        tb[s] = (uint64_t)((sb + m - 1) / m) + n_s * o;
    }
    u128 Df[8][8], Db[8][8];
    int has[8][8];
    memset(Df, 0, sizeof Df); memset(Db, 0, sizeof Db); memset(has, 0, sizeof has);
    for (int e = 0; e < c->E; e++) {
        int a = stage_of[c->e_src[e]], b = stage_of[c->e_dst[e]];
        if (a == b) continue;
        Df[a][b] += c->e_bf[e]; Db[a][b] += c->e_bb[e]; has[a][b] = 1;
    }
    free(stage_of);
    uint64_t cf[8][8], cb[8][8];
    for (int a = 0; a < M; a++)
        for (int b = 0; b < M; b++) {
            u128 den = (u128)m * c->link_bw;
            cf[a][b] = has[a][b] ? (uint64_t)((Df[a][b] * 1000000000000ULL + den - 1) / den) + c->link_lat : 0;
            cb[a][b] = has[a][b] ? (uint64_t)((Db[a][b] * 1000000000000ULL + den - 1) / den) + c->link_lat : 0;
        }
    uint64_t *F = calloc((size_t)M * m, 8), *B = calloc((size_t)M * m, 8);
#define FF(s, j) F[(size_t)(s) * m + (j)]
#define BB(s, j) B[(size_t)(s) * m + (j)]
    for (uint32_t j = 0; j < m; j++)
        for (int s = 0; s < M; s++) {
            uint64_t r = j > 0 ? FF(s, j - 1) : 0;
            for (int a = 0; a < s; a++)
                if (has[a][s] && FF(a, j) + cf[a][s] > r) r = FF(a, j) + cf[a][s];
            FF(s, j) = r + tf[s];
        }
    for (int64_t j = (int64_t)m - 1; j >= 0; j--)
        for (int s = M - 1; s >= 0; s--) {
            uint64_t r = (j == (int64_t)m - 1) ? FF(s, m - 1) : BB(s, j + 1);
            for (int b = s + 1; b < M; b++)
                if (has[s][b] && BB(b, j) + cb[s][b] > r) r = BB(b, j) + cb[s][b];
            BB(s, j) = r + tb[s];
        }
    uint64_t mk = 0;
    for (int s = 0; s < M; s++) if (BB(s, 0) > mk) mk = BB(s, 0);
#undef FF
#undef BB
    free(F); free(B);
    return mk;
}

uint64_t or_pipeline(const or_ctx *c, int M, const int32_t *cuts, uint32_t m) {
    return or_pipeline_ex(c, M, cuts, m, 0);
}

/* Exhaustive pipeline search: cut vectors in lexicographic order (rank r),
 * micro-batch counts micro[0..nm−1]; candidate index = r·nm + j.  Returns the
 * lexicographically smallest (makespan, index) over [begin, end).            */
or_best or_pipeline_search_ex(const or_ctx *c, int M, const uint32_t *micro, int nm,
                              uint64_t begin, uint64_t end, uint64_t o) {
    or_best best = { UINT64_MAX, UINT64_MAX };
    if (M < 1 || M > 8 || M > c->K || nm < 1) return best;
    /* start at the first rank touching [begin, end): unrank it (combinatorial
     * number system, lexicographic order of cut vectors from {1..K−1})      */
    uint64_t r = begin / (uint64_t)nm;
    int cuts[8];
    {
        u128 rank = r;
        int x = 1;
        for (int i = 0; i < M - 1; i++) {
            for (;;) {
                /* combinations with cuts[i] = x: choose the remaining M−2−i cuts
                 * from {x+1..K−1} */
                u128 cnt = 1;
                int n = c->K - 1 - x, k = M - 2 - i;
                if (k > n) cnt = 0;
                else for (int t = 1; t <= k; t++) cnt = cnt * (u128)(n - k + t) / (u128)t;
                if (rank < cnt) break;
                rank -= cnt;
                x++;
                if (x > c->K - 1) return best;       /* beyond the last combination */
            }
            cuts[i] = x++;
        }
    }
    for (;;) {
        for (int j = 0; j < nm; j++) {
            uint64_t idx = r * (uint64_t)nm + (uint64_t)j;
            if (idx >= begin && idx < end) {
                uint64_t mk = or_pipeline_ex(c, M, cuts, micro[j], o);
                if (mk < best.makespan || (mk == best.makespan && idx < best.index)) {
                    best.makespan = mk; best.index = idx;
                }
            }
        }
        /* next combination of M−1 cuts from {1..K−1} */
        int i = M - 2;
        while (i >= 0 && cuts[i] == c->K - 1 - (M - 2 - i)) i--;
        if (i < 0) break;
        cuts[i]++;
        for (int t = i + 1; t < M - 1; t++) cuts[t] = cuts[t - 1] + 1;
        r++;
        if (r * (uint64_t)nm >= end) break;
    }
    return best;
}

or_best or_pipeline_search(const or_ctx *c, int M, const uint32_t *micro, int nm, uint64_t begin, uint64_t end) {
    return or_pipeline_search_ex(c, M, micro, nm, begin, end, 0);
}

/* ------------------------------------------------------- O5 / O6 generators */
#define OR_GEN_GRAY 0
#define OR_GEN_RANDOM 1
#define OR_GEN_PERTURB 2

/* SplitMix64 finaliser (SURVEY §8(c) O6 [proposal]; the paper has no generator). */
uint64_t or_mix(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27; z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

static int ceil_log2(int M) { int b = 0; while ((1 << b) < M) b++; return b; }

static uint64_t word_at(uint64_t seed, uint64_t i, uint64_t Wd, uint64_t t) {
    return or_mix(seed + 0x9E3779B97F4A7C15ULL * (i * Wd + t + 1));
}

/* Writes placement d[0..K-1] (π positions) of candidate i.
 * GRAY   : O5, reflected M-ary Gray code of i.
 * RANDOM : O6, b = ⌈log2 M⌉ bits per op, P = 8·⌊8/b⌋ ops per SplitMix64
 *          word (64, 32, 16 for b = 1, 2, 3), d = (x·M) >> b; i = 0 is all
 *          zeros.
 * PERTURB: O6, one byte per op, 8 ops per word: op j flips iff
 *          u_j = byte (j mod 8) of word'(i, ⌊j/8⌋) < τ (probability τ/256).
 *          A flipped op moves, with y_j = byte (j mod 8) of word''(i, ⌊j/8⌋):
 *            M = 2      to 1 − base;
 *            M = 4, 8   to base XOR (y_j mod M), i.e. it is re-drawn
 *                       uniformly over the M devices (revision 3);
 *            other M    to (base + 1 + y_j mod (M−1)) mod M.
 *          i = 0 is the base.  word' uses seed_r ^ 0xD1B54A32D192ED03,
 *          word'' seed_r ^ 0x8CB92BA72F3D8DD7.
 * (Generator spec revision 3: word boundaries fall on 8-op groups, and the
 * power-of-two device counts re-draw by XOR; DESIGN.md §Generators.  The
 * paper has no generator; this is the shared spec.)                         */
void or_gen(int K, int M, int gen, uint64_t seed_r, uint32_t tau,
            const uint8_t *base, uint64_t i, uint8_t *d) {
    if (M == 1) { for (int j = 0; j < K; j++) d[j] = 0; return; }
    if (gen == OR_GEN_GRAY) {
        uint64_t *a = malloc(8 * (size_t)(K + 1));
        uint64_t x = i;
        for (int j = 0; j < K; j++) { a[j] = x % (uint64_t)M; x /= (uint64_t)M; }
        a[K] = 0;
        for (int j = 0; j < K; j++) {
            uint64_t par;
            if (M % 2 == 0) par = a[j + 1];
            else { par = 0; for (int t = j + 1; t <= K; t++) par += a[t]; }
            d[j] = (uint8_t)((par % 2 == 0) ? a[j] : (uint64_t)(M - 1) - a[j]);
        }
        free(a);
        return;
    }
    int b = ceil_log2(M);
    if (gen == OR_GEN_RANDOM) {
        if (i == 0) { for (int j = 0; j < K; j++) d[j] = 0; return; }
        uint64_t P = 8 * (uint64_t)(8 / b);
        uint64_t Wd = ((uint64_t)K + P - 1) / P;
        for (int j = 0; j < K; j++) {
            uint64_t w = word_at(seed_r, i, Wd, (uint64_t)j / P);
            uint64_t x = (w >> ((uint64_t)b * ((uint64_t)j % P))) & ((1ULL << b) - 1);
            d[j] = (uint8_t)((x * (uint64_t)M) >> b);
        }
        return;
    }
    /* PERTURB */
    if (i == 0) { for (int j = 0; j < K; j++) d[j] = base[j]; return; }
    uint64_t s1 = seed_r ^ 0xD1B54A32D192ED03ULL, s2 = seed_r ^ 0x8CB92BA72F3D8DD7ULL;
    uint64_t Wd = ((uint64_t)K + 7) / 8;
    for (int j = 0; j < K; j++) {
        uint64_t u = (word_at(s1, i, Wd, (uint64_t)j / 8) >> (8 * ((uint64_t)j % 8))) & 0xFF;
        if (u >= tau) { d[j] = base[j]; continue; }
        if (M == 2) { d[j] = (uint8_t)(1 - base[j]); continue; }
        uint64_t y = (word_at(s2, i, Wd, (uint64_t)j / 8) >> (8 * ((uint64_t)j % 8))) & 0xFF;
        if (M == 4 || M == 8) { d[j] = (uint8_t)(base[j] ^ (y % (uint64_t)M)); continue; }
        d[j] = (uint8_t)((base[j] + 1 + (y % (uint64_t)(M - 1))) % (uint64_t)M);
    }
}

/* O7 (one round): lexicographic min of (makespan, i) over candidates
 * i ∈ [begin, end) with seed_r and base (π order).                         */

or_best or_round(const or_ctx *c, int M, int gen, uint64_t seed_r, uint32_t tau,
                 const uint8_t *base, uint64_t begin, uint64_t end) {
    or_best best = { UINT64_MAX, UINT64_MAX };
    uint8_t *d = malloc((size_t)c->K);
    for (uint64_t i = begin; i < end; i++) {
        or_gen(c->K, M, gen, seed_r, tau, base, i, d);
        uint64_t mk = or_schedule(c, M, d);
        if (mk < best.makespan || (mk == best.makespan && i < best.index)) {
            best.makespan = mk; best.index = i;
        }
    }
    free(d);
    return best;
}

/* argmin over candidates [begin, end) of the EXACT makespan (NEXT f1),
 * lexicographic (makespan, index) as in O7                                   */
or_best or_round_exact(const or_ctx *c, int M, int gen, uint64_t seed_r, uint32_t tau,
                       const uint8_t *base, uint64_t begin, uint64_t end) {
    or_best best = { UINT64_MAX, UINT64_MAX };
    uint8_t *d = malloc((size_t)c->K + 1);
    for (uint64_t i = begin; i < end; i++) {
        or_gen(c->K, M, gen, seed_r, tau, base, i, d);
        uint64_t mk = or_exact(c, M, d);
        if (mk < best.makespan || (mk == best.makespan && i < best.index)) {
            best.makespan = mk; best.index = i;
        }
    }
    free(d);
    return best;
}

typedef struct {
    uint64_t best_makespan_ps, best_index, best_round, t1_ps, evaluated;
} or_result;

/* O7: full search.  PERTURB rounds: seed_r = seed + r; the base moves to the
 * round winner iff its makespan is strictly below the base's.  The reported
 * best is the first round that reached the final best makespan (R9 ties to
 * the smallest candidate index).  placement_orig receives the winner in
 * descriptor order.  base_orig (descriptor order) may be NULL (all zero).   */
int or_search(const or_ctx *c, int M, int gen, uint64_t seed, uint64_t count,
              uint32_t rounds, uint32_t tau, const uint8_t *base_orig,
              or_result *res, uint8_t *placement_orig) {
    int K = c->K;
    if (M < 1 || M > 8 || count < 1 || rounds < 1 || gen < 0 || gen > 2 || tau > 256) return OR_E_INVALID;
    if (c->nd && M > c->nd) return OR_E_INVALID;   /* devices 0..M−1 of the hardware graph */
    if (gen != OR_GEN_PERTURB && rounds != 1) return OR_E_INVALID;
    if (gen == OR_GEN_GRAY) {
        u128 space = 1;
        for (int j = 0; j < K && space <= ((u128)1 << 63); j++) space *= (u128)M;
        if (space > ((u128)1 << 63)) return OR_E_TOO_LARGE;
        if ((u128)count > space) return OR_E_INVALID;
    }
    uint8_t *base = calloc((size_t)K, 1), *d = malloc((size_t)K), *bestd = malloc((size_t)K);
    if (base_orig) for (int p = 0; p < K; p++) {
        base[p] = base_orig[c->pi[p]];
        if (base[p] >= M) { free(base); free(d); free(bestd); return OR_E_INVALID; }
    }
    or_best overall = { UINT64_MAX, UINT64_MAX };
    uint64_t best_round = 0;
    for (uint32_t r = 0; r < rounds; r++) {
        uint64_t seed_r = seed + r;
        or_best w = or_round(c, M, gen, seed_r, tau, base, 0, count);
        or_gen(K, M, gen, seed_r, tau, base, w.index, d);
        if (r == 0 || w.makespan < overall.makespan) {
            overall = w; best_round = r;
            memcpy(bestd, d, (size_t)K);
        }
        /* base of the next round: candidate 0 is the base, so the winner's
         * makespan is ≤ the base's; move iff strictly smaller              */
        uint64_t base_mk = or_schedule(c, M, base);
        if (w.makespan < base_mk) memcpy(base, d, (size_t)K);
    }
    res->best_makespan_ps = overall.makespan;
    res->best_index = overall.index;
    res->best_round = best_round;
    res->t1_ps = c->t1;
    res->evaluated = count * (uint64_t)rounds;
    if (placement_orig) for (int p = 0; p < K; p++) placement_orig[c->pi[p]] = bestd[p];
    free(base); free(d); free(bestd);
    if (overall.makespan == OR_INFEASIBLE_MAKESPAN) return OR_E_INFEASIBLE;
    return OR_OK;
}

/* ------------------------------------------------------ O8–O11 projection */
typedef struct {
    uint64_t dataset_items;            /* D  (§3) */
    uint32_t mini_batch;               /* B  (§3.1) */
    uint32_t n_knots;
    const uint64_t *knot_G, *knot_uepochs; /* E(G) curve, µ-epochs (Fig. 4) */
    uint64_t grad_bytes;               /* S for the ring all-reduce */
    uint64_t bw_intra_Bps, lat_intra_ps, bw_inter_Bps, lat_inter_ps;
    uint32_t node_size;                /* 0 => 8 */
    uint32_t ar_mode;                  /* 0 = EQ5 (paper Eq. 5), 1 = TIME */
    uint64_t t1_ps;                    /* T_1 */
    /* NEXT f4 */
    uint32_t n_accum, _pad;            /* accumulation factors a per cell; 0 => {1} */
    const uint32_t *accum;             /* PAPER.md:251 delayed gradient update      */
    const uint64_t *shard_bytes;       /* [nM][8] per-device gradient shards, or NULL */
} or_scenario;

typedef struct { uint64_t C_lo, C_hi, step_ps, steps, uepochs; uint32_t feasible, accum; } or_cell;

static int bitlen128(u128 x) { int n = 0; while (x) { n++; x >>= 1; } return n; }

/* O8: ring all-reduce of S bytes over n workers (PAPER.md:120 ring all-reduce;
 * PAPER.md:171 slower inter-node links; reading R10):
 *   AR(n,S) = 0 if n = 1, else ⌈2(n−1)·S·10^12 / (n·BW)⌉ + 2(n−1)·α,
 *   tier = intra if the cell's device count ≤ node_size else inter;
 *   a tier with BW = 0 is "AR off" (SE ≡ 1).                    */
static int or_ar_S(const or_scenario *s, uint64_t n, uint64_t n_devices, uint64_t S, u128 *out) {
    *out = 0;
    if (n <= 1) return OR_OK;
    uint64_t node = s->node_size ? s->node_size : 8;
    uint64_t bw = (n_devices <= node) ? s->bw_intra_Bps : s->bw_inter_Bps;
    uint64_t al = (n_devices <= node) ? s->lat_intra_ps : s->lat_inter_ps;
    if (bw == 0) return OR_OK;
    u128 num = (u128)2 * (n - 1);
    if (bitlen128(num) + bitlen128(S) + 40 > 127) return OR_E_RANGE;
    num = num * S * (u128)1000000000000ULL;
    u128 den = (u128)n * bw;
    u128 q = num / den + (num % den ? 1 : 0);
    *out = q + (u128)2 * (n - 1) * al;
    return OR_OK;
}

int or_ar(const or_scenario *s, uint64_t n, uint64_t n_devices, u128 *out) {
    return or_ar_S(s, n, n_devices, s->grad_bytes, out);
}

uint64_t or_ar64(const or_scenario *s, uint64_t n, uint64_t n_devices, int *rc) {
    u128 a; *rc = or_ar(s, n, n_devices, &a);
    if (*rc == OR_OK && (a >> 64)) *rc = OR_E_RANGE;
    return (uint64_t)a;
}

/* O9: E(G) from the knots (Fig. 4 shape; reading R12): exact at knots,
 * floor of the linear interpolation in G between knots, infeasible outside. */
int or_epochs(const or_scenario *s, uint64_t G, uint64_t *E) {
    uint32_t n = s->n_knots;
    if (n == 0 || G < s->knot_G[0] || G > s->knot_G[n - 1]) return 0;
    for (uint32_t i = 0; i < n; i++) if (s->knot_G[i] == G) { *E = s->knot_uepochs[i]; return 1; }
    for (uint32_t i = 0; i + 1 < n; i++) {
        uint64_t g0 = s->knot_G[i], g1 = s->knot_G[i + 1];
        if (g0 < G && G < g1) {
            u128 num = (u128)s->knot_uepochs[i] * (g1 - G) + (u128)s->knot_uepochs[i + 1] * (G - g0);
            *E = (uint64_t)(num / (g1 - g0));
            return 1;
        }
    }
    return 0;
}

static int validate_scenario(const or_scenario *s) {
    if (s->mini_batch == 0 || s->dataset_items == 0 || s->t1_ps == 0 || s->ar_mode > 1) return OR_E_INVALID;
    if (s->n_accum > 32 || (s->n_accum && !s->accum)) return OR_E_INVALID;
    for (uint32_t j = 0; j < s->n_accum; j++) if (s->accum[j] == 0) return OR_E_INVALID;
    if (s->n_knots == 0 || !s->knot_G || !s->knot_uepochs) return OR_E_INVALID;
    for (uint32_t i = 0; i < s->n_knots; i++) {
        if (s->knot_uepochs[i] == 0) return OR_E_INVALID;
        if (i > 0 && s->knot_G[i] <= s->knot_G[i - 1]) return OR_E_INVALID;
        if (i > 0) {
            uint64_t em = s->knot_uepochs[i] > s->knot_uepochs[i - 1] ? s->knot_uepochs[i] : s->knot_uepochs[i - 1];
            if (bitlen128(em) + bitlen128(s->knot_G[i] - s->knot_G[i - 1]) + 1 > 127) return OR_E_RANGE;
        }
    }
    return OR_OK;
}

/* O10: one cell (M, N).  Eq. 1 C = T×S×E; S = ⌈D/G⌉
 * (reading R14); G = W·B·a with W = N/M workers
 * and a mini-batches accumulated per step (NEXT f4, PAPER.md:251 delayed
 * gradient update; a = 1 unless the scenario offers more);
 * EQ5 (Eq. 5, reading R11): T = ⌊(a·T_1 + AR(W))·T_M / T_1⌋;
 * TIME: T = a·T_M + AR(W).  AR(W) all-reduces grad_bytes, or with per-device
 * shards (NEXT f4, reading R24) the slowest shard: max_d AR(W, S_d).
 * The cell keeps the a with the smallest C (ties → the earlier a in the list).
 * M ∤ N => infeasible (R15).                                                  */
int or_cell_compute_ex(const or_scenario *s, uint32_t M, uint64_t T_M, uint32_t N, const uint64_t *shard,
                       or_cell *cell) {
    memset(cell, 0, sizeof *cell);
    if (M == 0 || N == 0) return OR_E_INVALID;
    if (N % M != 0) return OR_OK;
    uint64_t W = N / M;
    u128 A = 0;
    if (shard) {
        for (uint32_t d = 0; d < M && d < 8; d++) {
            u128 Ad;
            int rc = or_ar_S(s, W, N, shard[d], &Ad);
            if (rc) return rc;
            if (Ad > A) A = Ad;
        }
    } else {
        int rc = or_ar(s, W, N, &A);
        if (rc) return rc;
    }
    uint32_t na = s->n_accum ? s->n_accum : 1;
    for (uint32_t j = 0; j < na; j++) {
        uint64_t a = s->n_accum ? s->accum[j] : 1;
        u128 G = (u128)W * s->mini_batch * a;
        uint64_t E;
        if (G >> 64) continue;
        if (!or_epochs(s, (uint64_t)G, &E)) continue;
        u128 T;
        if (s->ar_mode == 0) {
            u128 x = (u128)a * s->t1_ps + A;
            if (bitlen128(x) + bitlen128(T_M) > 127) return OR_E_RANGE;
            T = x * T_M / s->t1_ps;
        } else {
            T = (u128)a * T_M + A;
        }
        if (T >> 64) return OR_E_RANGE;
        uint64_t steps = (uint64_t)((s->dataset_items + (uint64_t)G - 1) / (uint64_t)G);
        if (bitlen128(T) + bitlen128(steps) + bitlen128(E) > 127) return OR_E_RANGE;
        u128 C = T * steps * E;
        if (!cell->feasible || C < (((u128)cell->C_hi << 64) | cell->C_lo)) {
            cell->C_lo = (uint64_t)C; cell->C_hi = (uint64_t)(C >> 64);
            cell->step_ps = (uint64_t)T; cell->steps = steps; cell->uepochs = E; cell->feasible = 1;
            cell->accum = (uint32_t)a;
        }
    }
    return OR_OK;
}

int or_cell_compute(const or_scenario *s, uint32_t M, uint64_t T_M, uint32_t N, or_cell *cell) {
    return or_cell_compute_ex(s, M, T_M, N, NULL, cell);
}

/* cells[m*N_max + (N-1)] */
int or_project(const or_scenario *s, int nM, const uint32_t *Ms, const uint64_t *T_M,
               uint32_t N_max, or_cell *cells) {
    int rc = validate_scenario(s);
    if (rc) return rc;
    if (nM < 1 || nM > 8 || N_max < 1 || N_max > 65536) return OR_E_INVALID;
    for (int m = 0; m < nM; m++) if (Ms[m] == 0 || T_M[m] == 0) return OR_E_INVALID;
    for (int m = 0; m < nM; m++)
        for (uint32_t N = 1; N <= N_max; N++) {
            rc = or_cell_compute_ex(s, Ms[m], T_M[m], N, s->shard_bytes ? s->shard_bytes + 8 * (size_t)m : NULL,
                                    &cells[(size_t)m * N_max + (N - 1)]);
            if (rc) return rc;
        }
    return OR_OK;
}

typedef struct {
    uint32_t n_star, m_at_n_star;
    uint32_t n_star_M[8], persistent_M[8];
    uint32_t n_star_vs_best_dp;
} or_crossover_result;

static u128 cellC(const or_cell *c) { return ((u128)c->C_hi << 64) | c->C_lo; }

/* O11: crossover (Eq. 6, strict ">", reading R16; §5
 * PAPER.md:310–317).  best_m (optional, length N_max) receives the M with the
 * smallest C at each N (ties → smaller M), 0 if none.        */
int or_crossover(const or_cell *cells, int nM, const uint32_t *Ms, uint32_t N_max,
                 or_crossover_result *res, uint32_t *best_m) {
    memset(res, 0, sizeof *res);
    int m1 = -1;
    for (int m = 0; m < nM; m++) if (Ms[m] == 1) m1 = m;
    if (m1 < 0 || nM < 1 || nM > 8 || N_max < 1) return OR_E_INVALID;
    const or_cell *dp = cells + (size_t)m1 * N_max;
    for (int m = 0; m < nM; m++) {
        if (Ms[m] == 1) continue;
        const or_cell *hy = cells + (size_t)m * N_max;
        uint32_t ns = 0;
        for (uint32_t N = 1; N <= N_max && !ns; N++) {
            const or_cell *a = &hy[N - 1], *b = &dp[N - 1];
            if (a->feasible && b->feasible && cellC(a) < cellC(b)) ns = N;
        }
        res->n_star_M[m] = ns;
        if (ns) {
            uint32_t pers = 1;
            for (uint32_t N = ns; N <= N_max; N++) {
                const or_cell *a = &hy[N - 1], *b = &dp[N - 1];
                if (a->feasible && b->feasible && !(cellC(a) < cellC(b))) pers = 0;
            }
            res->persistent_M[m] = pers;
            if (res->n_star == 0 || ns < res->n_star) res->n_star = ns;
        }
    }
    if (res->n_star) {
        uint32_t N = res->n_star;
        int bm = -1;
        for (int m = 0; m < nM; m++) {
            const or_cell *a = &cells[(size_t)m * N_max + (N - 1)];
            if (!a->feasible) continue;
            if (bm < 0 || cellC(a) < cellC(&cells[(size_t)bm * N_max + (N - 1)]) ||
                (cellC(a) == cellC(&cells[(size_t)bm * N_max + (N - 1)]) && Ms[m] < Ms[bm])) bm = m;
        }
        res->m_at_n_star = Ms[bm];
    }
    /* n_star_vs_best_dp: min N with min_M C(M,N) < min_{N'≤N} C(1,N')
     * ("speedup over the best performing scale of DP-only");
     * N with no feasible DP cell at or below it are skipped.                 */
    int have_dp = 0; u128 best_dp = 0;
    for (uint32_t N = 1; N <= N_max; N++) {
        if (dp[N - 1].feasible && (!have_dp || cellC(&dp[N - 1]) < best_dp)) { best_dp = cellC(&dp[N - 1]); have_dp = 1; }
        int bm = -1;
        for (int m = 0; m < nM; m++) {
            const or_cell *a = &cells[(size_t)m * N_max + (N - 1)];
            if (!a->feasible) continue;
            if (bm < 0 || cellC(a) < cellC(&cells[(size_t)bm * N_max + (N - 1)]) ||
                (cellC(a) == cellC(&cells[(size_t)bm * N_max + (N - 1)]) && Ms[m] < Ms[bm])) bm = m;
        }
        if (best_m) best_m[N - 1] = bm < 0 ? 0 : Ms[bm];
        if (!res->n_star_vs_best_dp && have_dp && bm >= 0 &&
            cellC(&cells[(size_t)bm * N_max + (N - 1)]) < best_dp) res->n_star_vs_best_dp = N;
    }
    return OR_OK;
}
