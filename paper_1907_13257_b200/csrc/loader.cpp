// loader.cpp — pp_load_dfg: validation, π, edge costs, forward+backward
// schedule records, liveness slots, packed shared-memory image, upload.
//
// PAPER.md:350 (§6) defines the DFG (K, E, Δ(k), M(k), D(e))
// the edge delay Δ_e = Σ_l C_el·(D(e)/B(l) + L(l)), here one NVSwitch hop (R4):
// c(e) = ⌈D(e)·10^12 / BW⌉ + L in integer ps.  π is Kahn's algorithm with the
// smallest external id first (R3).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <queue>
#include <unordered_set>

#include "internal.h"

namespace pp {

typedef unsigned __int128 u128;

static int fail(int code, const std::string &msg) {
    set_error(msg);
    return code;
}

// Kahn with a min-heap keyed by external id.  On a cycle, names one cycle.
static int topo_order(int K, const std::vector<int64_t> &id, const std::vector<int32_t> &src,
                      const std::vector<int32_t> &dst, std::vector<int32_t> &pi) {
    std::vector<int> indeg(K, 0);
    std::vector<std::vector<int>> succ(K), pred(K);
    for (size_t e = 0; e < src.size(); e++) {
        indeg[dst[e]]++;
        succ[src[e]].push_back(dst[e]);
        pred[dst[e]].push_back(src[e]);
    }
    typedef std::pair<int64_t, int> Item;
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
    for (int k = 0; k < K; k++)
        if (indeg[k] == 0) heap.push(Item(id[k], k));
    std::vector<char> done(K, 0);
    pi.clear();
    while (!heap.empty()) {
        int k = heap.top().second;
        heap.pop();
        done[k] = 1;
        pi.push_back(k);
        for (int v : succ[k])
            if (--indeg[v] == 0) heap.push(Item(id[v], v));
    }
    if ((int)pi.size() == K) return PP_OK;
    // every unfinished op has an unfinished predecessor: walk back until repeat
    int v = 0;
    while (done[v]) v++;
    std::vector<int> seen(K, -1);
    for (int step = 0; seen[v] < 0; step++) {
        seen[v] = step;
        for (int u : pred[v])
            if (!done[u]) { v = u; break; }
    }
    std::string msg = "cycle:";
    int start = v;
    do {
        msg += " " + std::to_string(id[v]);
        for (int u : pred[v])
            if (!done[u]) { v = u; break; }
    } while (v != start);
    return fail(PP_E_CYCLE, msg);
}

// Delay-shortest route cost from device a to every node for a payload
// (general hardware graph, pp_hw_desc): binary-heap Dijkstra, u128.
static void route_costs(const pp_hw_desc *hw, uint64_t bytes, int src, std::vector<u128> &dist) {
    const int V = hw->num_devices + hw->num_routers;
    const u128 INF = ~(u128)0;
    dist.assign(V, INF);
    typedef std::pair<u128, int> Item;
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
    dist[src] = 0;
    heap.push(Item(0, src));
    while (!heap.empty()) {
        Item it = heap.top();
        heap.pop();
        if (it.first != dist[it.second]) continue;
        const int u = it.second;
        for (int l = 0; l < hw->num_links; l++) {
            int v;
            if (hw->link_a[l] == u) v = hw->link_b[l];
            else if (hw->link_b[l] == u) v = hw->link_a[l];
            else continue;
            const u128 w = ((u128)bytes * 1000000000000ull + hw->link_bw_Bps[l] - 1) / hw->link_bw_Bps[l] +
                           hw->link_lat_ps[l];
            if (it.first + w < dist[v]) {
                dist[v] = it.first + w;
                heap.push(Item(dist[v], v));
            }
        }
    }
}

// plan / plan_tier non-null: a dry run (pp_plan_dfg) — validation, π, the
// slot allocation and the tier, reported without touching a device.
int load_dfg(const pp_dfg_desc *d, const pp_link_desc *link, const pp_hw_desc *hw, int cuda_device,
             pp_dfg **out, pp_dfg_info *plan, int32_t *plan_tier) {
    const bool dry = plan != nullptr;
    if (!out && !dry) return fail(PP_E_INVALID, "out is NULL");
    if (out) *out = nullptr;
    if (dry && !plan_tier) return fail(PP_E_INVALID, "tier is NULL");
    if (!d || (!link && !hw)) return fail(PP_E_INVALID, "desc or link is NULL");
    if (hw) {
        if (hw->num_devices < 1 || hw->num_devices > 8 || hw->num_routers < 0 || hw->num_links < 0 ||
            (hw->num_links > 0 && (!hw->link_a || !hw->link_b || !hw->link_bw_Bps || !hw->link_lat_ps)))
            return fail(PP_E_INVALID, "invalid hardware graph sizes");
        const int V = hw->num_devices + hw->num_routers;
        for (int l = 0; l < hw->num_links; l++)
            if (hw->link_a[l] < 0 || hw->link_a[l] >= V || hw->link_b[l] < 0 || hw->link_b[l] >= V ||
                hw->link_a[l] == hw->link_b[l] || hw->link_bw_Bps[l] == 0)
                return fail(PP_E_INVALID, "invalid link " + std::to_string(l));
    }
    const int K = d->num_ops, E = d->num_edges;
    if (K < 1 || E < 0 || !d->fwd_ps || !d->bwd_ps ||
        (E > 0 && (!d->edge_src || !d->edge_dst || !d->edge_fwd_bytes)))
        return fail(PP_E_INVALID, "invalid sizes or null arrays");
    if (!hw && link->link_bw_Bps == 0) return fail(PP_E_INVALID, "link bandwidth must be > 0");
    if (K > 65535) return fail(PP_E_TOO_LARGE, "more than 65535 ops");

    std::vector<int64_t> id(K);
    std::unordered_set<int64_t> ids;
    for (int k = 0; k < K; k++) {
        id[k] = d->op_id ? d->op_id[k] : k;
        if (id[k] < 0) return fail(PP_E_INVALID, "negative op id");
        if (!ids.insert(id[k]).second) return fail(PP_E_INVALID, "duplicate op id " + std::to_string(id[k]));
    }
    std::vector<int32_t> src(E), dst(E);
    for (int e = 0; e < E; e++) {
        src[e] = d->edge_src[e];
        dst[e] = d->edge_dst[e];
        if (src[e] < 0 || src[e] >= K || dst[e] < 0 || dst[e] >= K)
            return fail(PP_E_INVALID, "dangling edge endpoint at edge " + std::to_string(e));
        if (src[e] == dst[e]) return fail(PP_E_INVALID, "self edge at edge " + std::to_string(e));
    }
    std::vector<int32_t> pi;
    int rc = topo_order(K, id, src, dst, pi);
    if (rc) return rc;
    std::vector<int32_t> pos(K);
    for (int p = 0; p < K; p++) pos[pi[p]] = p;

    // edge costs and the 2^61 time bound (times are tagged as 8·t + device)
    std::vector<uint64_t> cf(E), cb(E);
    u128 bound = 0;
    for (int k = 0; k < K; k++) bound += (u128)d->fwd_ps[k] + d->bwd_ps[k];
    const u128 t1 = bound;
    // hardware graph: cost of every ordered device pair, classes of pairs
    const int nd = hw ? hw->num_devices : 0;
    std::vector<uint64_t> hcf, hcb;           // [e][a][b]
    std::vector<int> cls(64, 0);              // class of (a, b); 0 for a == b
    int ncls = 1;
    if (hw) {
        hcf.assign((size_t)E * nd * nd, 0);
        hcb.assign((size_t)E * nd * nd, 0);
        std::vector<u128> dist;
        for (int a = 0; a < nd; a++) {
            route_costs(hw, 0, a, dist);
            for (int b = 0; b < nd; b++)
                if (dist[b] == ~(u128)0) return fail(PP_E_INVALID, "devices not connected");
        }
        for (int e = 0; e < E; e++) {
            uint64_t bf = d->edge_fwd_bytes[e];
            uint64_t bb = d->edge_bwd_bytes ? d->edge_bwd_bytes[e] : bf;
            u128 mf = 0, mb = 0;
            for (int dir = 0; dir < 2; dir++)
                for (int a = 0; a < nd; a++) {
                    route_costs(hw, dir ? bb : bf, a, dist);
                    for (int b = 0; b < nd; b++) {
                        if (a == b) continue;
                        if (dist[b] >> 64) return fail(PP_E_RANGE, "edge cost overflow");
                        (dir ? hcb : hcf)[((size_t)e * nd + a) * nd + b] = (uint64_t)dist[b];
                        u128 &m = dir ? mb : mf;
                        if (dist[b] > m) m = dist[b];
                    }
                }
            bound += mf + mb;
            if (bound >> 61) return fail(PP_E_RANGE, "time bound >= 2^61 ps");
        }
        // pairs with equal costs on every edge and direction share a class
        std::vector<std::vector<uint64_t>> reps;
        for (int a = 0; a < nd; a++)
            for (int b = 0; b < nd; b++) {
                if (a == b) continue;
                std::vector<uint64_t> v(2 * (size_t)E);
                for (int e = 0; e < E; e++) {
                    v[2 * e] = hcf[((size_t)e * nd + a) * nd + b];
                    v[2 * e + 1] = hcb[((size_t)e * nd + a) * nd + b];
                }
                size_t c = 0;
                while (c < reps.size() && reps[c] != v) c++;
                if (c == reps.size()) reps.push_back(v);
                cls[a * 8 + b] = (int)c + 1;
            }
        ncls = (int)reps.size() + 1;
    } else {
        for (int e = 0; e < E; e++) {
            uint64_t bf = d->edge_fwd_bytes[e];
            uint64_t bb = d->edge_bwd_bytes ? d->edge_bwd_bytes[e] : bf;
            u128 qf = ((u128)bf * 1000000000000ull + link->link_bw_Bps - 1) / link->link_bw_Bps + link->link_lat_ps;
            u128 qb = ((u128)bb * 1000000000000ull + link->link_bw_Bps - 1) / link->link_bw_Bps + link->link_lat_ps;
            bound += qf + qb;
            if ((qf >> 64) || (qb >> 64) || (bound >> 61)) return fail(PP_E_RANGE, "time bound >= 2^61 ps");
            cf[e] = (uint64_t)qf;
            cb[e] = (uint64_t)qb;
        }
    }
    if (bound >> 61) return fail(PP_E_RANGE, "time bound >= 2^61 ps");
    if (hw && (bound >> 49)) return fail(PP_E_RANGE, "hardware-graph mode needs every time < 2^49 ps");

    // adjacency by π position
    std::vector<std::vector<int>> in_e(K), out_e(K);
    for (int e = 0; e < E; e++) {
        in_e[pos[dst[e]]].push_back(e);
        out_e[pos[src[e]]].push_back(e);
    }

    // ---- inputs of every step.  K8 = K padded to a multiple of 8 (no-op pads
    // at π positions p ≥ K).  Value ids: step s produces value s (forward
    // finish time of p = s, or backward finish time of p = 2K8−1−s); −1 = zero.
    const int K8 = (K + 7) / 8 * 8;
    const int S = 2 * K8;
    // (value id, edge code): code = 2·e + [backward], −1 for a zero-cost input
    std::vector<std::vector<std::pair<int, int64_t>>> inputs(S);
    for (int s = 0; s < S; s++) {
        const bool fwd = s < K8;
        const int p = fwd ? s : S - 1 - s;
        auto &in = inputs[s];
        if (p >= K) {
            in.push_back({-1, -1});                      // pad
        } else if (fwd) {
            for (int e : in_e[p]) in.push_back({pos[src[e]], 2 * (int64_t)e});
            if (in.empty()) in.push_back({-1, -1});
        } else {
            for (int e : out_e[p]) in.push_back({S - 1 - pos[dst[e]], 2 * (int64_t)e + 1});
            if (out_e[p].empty()) in.push_back({p, -1});  // sink: waits for its own forward (R1)
        }
    }
    // register forwarding: an input produced by the previous step goes first
    // and is read from a register instead of shared memory
    std::vector<char> fwd_first(S, 0);
    for (int s = 1; s < S; s++) {
        auto &in = inputs[s];
        for (size_t j = 0; j < in.size(); j++)
            if (in[j].first == s - 1) {
                std::swap(in[0], in[j]);
                fwd_first[s] = 1;
                break;
            }
    }
    // liveness over the remaining (shared-memory) reads
    std::vector<int> last(S, -1);
    for (int s = 0; s < S; s++)
        for (size_t j = 0; j < inputs[s].size(); j++) {
            const int v = inputs[s][j].first;
            if (v < 0 || (j == 0 && fwd_first[s])) continue;
            last[v] = std::max(last[v], s);
        }
    // linear-scan slot allocation in step order; a slot whose value is last
    // read at step s is reusable for the output of step s itself (the kernel
    // reads all inputs of a step before it writes the output)
    std::vector<int> slot(S, -1);
    std::vector<std::vector<int>> expire(S);
    std::vector<int> free_slots;               // min-heap of free slot ids
    int nslots = 0;
    for (int s = 0; s < S; s++) {
        for (int sl : expire[s]) {
            free_slots.push_back(sl);
            std::push_heap(free_slots.begin(), free_slots.end(), std::greater<int>());
        }
        if (last[s] < 0) continue;             // never read from shared memory: no store
        int sl;
        if (free_slots.empty()) sl = nslots++;
        else {
            std::pop_heap(free_slots.begin(), free_slots.end(), std::greater<int>());
            sl = free_slots.back();
            free_slots.pop_back();
        }
        slot[s] = sl;
        expire[last[s]].push_back(sl);
    }
    const int W = nslots;
    const uint32_t zero_off = (uint32_t)W * kSlotUnit;   // slot W always holds 0
    if (W + 1 > 4096) return fail(PP_E_TOO_LARGE, "too many live slots");

    // ---- arithmetic: exact integer ps in doubles when every time is < 2^49
    // (device tag in the 3 low mantissa bits), else tagged u64 (8·t + device)
    bool f64 = (bound >> 49) == 0;
    if (const char *a = getenv("PP_ARITH")) {
        if (!strcmp(a, "int64")) f64 = false;
    }
    if (hw) f64 = true;   // the class-cost rows are f64-encoded

    // ---- tier: the shared-memory tier needs the image plus
    // at least 4 warps of lane state ((W + 1 + 8) slots × 256 B at one
    // placement per lane, M ≤ 8) within the SM's shared memory; otherwise the
    // DFG runs on the global-state tier (search_big_kernel), as does a DFG
    // whose time bound needs tagged u64 (≥ 2^49 ps; the shared tier is built
    // for tagged f64 only).  PP_TIER=global forces that tier (tests).
    size_t n_extra_all = 0;
    for (int s = 0; s < S; s++) n_extra_all += inputs[s].size() - 1;
    const size_t image_est = ((sizeof(OpRec) * S + sizeof(ExtraRec) * n_extra_all + 13ull * K8 + 15) & ~size_t(15));
    bool big = image_est > (size_t)kMaxImageBytes ||
               ((image_est + 127) & ~size_t(127)) + 4ull * ((size_t)W + 9) * kSlotUnit > (size_t)kTierSmemBytes;
    if (const char *t = getenv("PP_TIER")) {
        if (!strcmp(t, "global")) big = true;
    }
    if (!f64 && !hw) big = true;   // the shared tier is built for tagged f64 only
    if (big && hw) return fail(PP_E_TOO_LARGE, "hardware graphs need the shared-memory tier (image + 4 warps of lane state within 200 KB)");
    auto enc = [&](uint64_t ps) -> uint64_t {
        if (!f64) return 8ull * ps;
        double x = (double)ps;   // exact: ps < 2^49
        uint64_t bits;
        memcpy(&bits, &x, 8);
        return bits;
    };

    // ---- records: first input inlined in the op record, the rest as extras.
    // Uniform link: the record holds the encoded cost.  Hardware graph: it
    // holds the byte offset of the input's cost row (one entry per class).
    std::vector<OpRec> ops(S);
    std::vector<ExtraRec> xr;
    std::vector<uint64_t> rows;                 // hardware graph: ncls entries per distinct input
    std::map<int64_t, uint32_t> row_of;                  // edge code -> row index (memo)
    std::map<std::vector<uint64_t>, uint32_t> row_idx;   // row contents -> row index (dedupe)
    auto cost_field = [&](int64_t code) -> uint64_t {
        if (!hw) {
            if (code < 0) return enc(0);
            return enc((code & 1) ? cb[code >> 1] : cf[code >> 1]);
        }
        auto it = row_of.find(code);
        if (it != row_of.end()) return it->second;   // patched to a byte offset below
        std::vector<uint64_t> row(ncls, enc(0));
        if (code >= 0) {
            const int e = (int)(code >> 1);
            const auto &h = (code & 1) ? hcb : hcf;
            for (int a = 0; a < nd; a++)
                for (int b = 0; b < nd; b++)   // any pair of a class has the same cost
                    if (a != b) row[cls[a * 8 + b]] = enc(h[((size_t)e * nd + a) * nd + b]);
        }
        auto r = row_idx.find(row);
        uint32_t idx;
        if (r != row_idx.end()) {
            idx = r->second;
        } else {   // edges with equal payloads share one row
            idx = (uint32_t)(rows.size() / ncls);
            rows.insert(rows.end(), row.begin(), row.end());
            row_idx.emplace(std::move(row), idx);
        }
        row_of.emplace(code, idx);
        return idx;
    };
    auto src_off = [&](int v) -> uint32_t { return v < 0 ? zero_off : (uint32_t)slot[v] * kSlotUnit; };
    for (int s = 0; s < S; s++) {
        const bool fwd = s < K8;
        const int p = fwd ? s : S - 1 - s;
        const auto &in = inputs[s];
        OpRec &o = ops[s];
        o.cost8 = p < K ? enc(fwd ? d->fwd_ps[pi[p]] : d->bwd_ps[pi[p]]) : enc(0);
        o.c8 = cost_field(in[0].second);
        o.src_off = fwd_first[s] ? kFromPrev : src_off(in[0].first);
        o.out_off = slot[s] < 0 ? kNoStore : (uint32_t)slot[s] * kSlotUnit;
        const uint32_t n_extra = (uint32_t)in.size() - 1;
        if (n_extra > 0xFFFF) return fail(PP_E_TOO_LARGE, "op with more than 65536 inputs");
        o.ctrl = (fwd_first[s] && n_extra == 0) ? 0u : (0x10000u | n_extra);
        o.base = 0;
        for (size_t q = 1; q < in.size(); q++) xr.push_back(ExtraRec{cost_field(in[q].second), src_off(in[q].first), 0});
    }
    size_t off_extra = sizeof(OpRec) * S;
    size_t off_mem = off_extra + sizeof(ExtraRec) * xr.size();
    size_t off_orig = off_mem + 8ull * K8;
    size_t off_hgw = off_orig + 4ull * K8;
    size_t off_cls = (off_hgw + (size_t)K8 + 15) & ~size_t(15);
    size_t off_rows = off_cls + (hw ? 64 : 0);
    size_t bytes = off_rows + 8ull * rows.size();
    bytes = (bytes + 15) & ~size_t(15);
    if (hw) {   // row indices -> byte offsets
        const uint64_t row_bytes = 8ull * ncls;
        for (auto &o : ops) o.c8 = off_rows + o.c8 * row_bytes;
        for (auto &x : xr) x.c8 = off_rows + x.c8 * row_bytes;
    }
    if (!big && bytes > (size_t)kMaxImageBytes) return fail(PP_E_TOO_LARGE, "DFG image exceeds 96 KB of shared memory");
    if (bytes >= (size_t)1 << 31) return fail(PP_E_TOO_LARGE, "DFG image exceeds 2 GB");
    if (dry) {
        plan->num_ops = K;
        plan->num_edges = E;
        plan->num_slots = W;
        plan->image_bytes = (int32_t)bytes;
        plan->t1_ps = (uint64_t)t1;
        uint64_t gb = 0;
        if (d->param_bytes)
            for (int k = 0; k < K; k++) gb += d->param_bytes[k];
        plan->grad_bytes = gb;
        *plan_tier = big ? PP_TIER_GLOBAL : PP_TIER_SHARED;
        return PP_OK;
    }

    pp_dfg *g = new pp_dfg();
    g->device = cuda_device;
    g->K = K;
    g->K8 = K8;
    g->E = E;
    g->W = W;
    g->f64 = f64;
    g->big = big;
    g->t1 = (uint64_t)t1;
    g->cap = hw ? hw->dev_mem_cap_bytes : link->dev_mem_cap_bytes;
    g->hw = hw != nullptr;
    g->nd = nd;
    g->off_cls = (uint32_t)off_cls;
    if (link) {
        g->link_bw = link->link_bw_Bps;
        g->link_lat = link->link_lat_ps;
    }
    g->e_src.resize(E); g->e_dst.resize(E); g->e_bf.resize(E); g->e_bb.resize(E);
    for (int e = 0; e < E; e++) {
        g->e_src[e] = pos[src[e]];
        g->e_dst[e] = pos[dst[e]];
        g->e_bf[e] = d->edge_fwd_bytes[e];
        g->e_bb[e] = d->edge_bwd_bytes ? d->edge_bwd_bytes[e] : d->edge_fwd_bytes[e];
    }
    g->fwd.resize(K); g->bwd.resize(K); g->mem.resize(K);
    for (int p = 0; p < K; p++) {
        g->fwd[p] = d->fwd_ps[pi[p]];
        g->bwd[p] = d->bwd_ps[pi[p]];
        g->mem[p] = d->mem_bytes ? d->mem_bytes[pi[p]] : 0;
    }
    g->grad_bytes = 0;
    g->param.assign(K, 0);
    if (d->param_bytes)
        for (int k = 0; k < K; k++) g->param[k] = d->param_bytes[k];
    if (d->param_bytes)
        for (int k = 0; k < K; k++) g->grad_bytes += d->param_bytes[k];
    g->pi = pi;
    g->pos = pos;
    g->image.assign(bytes, 0);
    memcpy(g->image.data(), ops.data(), sizeof(OpRec) * S);
    if (!xr.empty()) memcpy(g->image.data() + off_extra, xr.data(), sizeof(ExtraRec) * xr.size());
    for (int p = 0; p < K8; p++) {
        uint64_t m = (p < K && d->mem_bytes) ? d->mem_bytes[pi[p]] : 0;
        memcpy(g->image.data() + off_mem + 8ull * p, &m, 8);
        uint32_t o = p < K ? (uint32_t)pi[p] : 0u;
        memcpy(g->image.data() + off_orig + 4ull * p, &o, 4);
    }
    if (hw) {
        for (int i = 0; i < 64; i++) g->image[off_cls + i] = (uint8_t)cls[i];
        memcpy(g->image.data() + off_rows, rows.data(), 8 * rows.size());
    }
    g->off_extra = (uint32_t)off_extra;
    g->off_mem = (uint32_t)off_mem;
    g->off_orig = (uint32_t)off_orig;
    g->off_hgw = (uint32_t)off_hgw;
    g->image_bytes = (uint32_t)bytes;
    g->base_bytes = (uint32_t)((K + 15) & ~15);

    // ---- cost rows shared by the exact-schedule and EFT images: plain u64 ps
    // per device-pair class, deduplicated by content; row 0 is all zero
    const int xcls = hw ? ncls : 2;
    std::vector<uint8_t> xc(64, 0);
    for (int a = 0; a < 8; a++)
        for (int b = 0; b < 8; b++) xc[a * 8 + b] = hw ? (uint8_t)cls[a * 8 + b] : (uint8_t)(a != b);
    std::vector<uint64_t> xrows(xcls, 0);
    std::map<std::vector<uint64_t>, uint32_t> xrow_idx;
    xrow_idx.emplace(std::vector<uint64_t>(xcls, 0), 0u);
    auto xrow = [&](int e, bool bwd) -> uint32_t {
        std::vector<uint64_t> r(xcls, 0);
        if (hw) {
            const auto &h = bwd ? hcb : hcf;
            for (int a = 0; a < nd; a++)
                for (int b = 0; b < nd; b++)
                    if (a != b) r[cls[a * 8 + b]] = h[((size_t)e * nd + a) * nd + b];
        } else {
            r[1] = bwd ? cb[e] : cf[e];
        }
        auto it = xrow_idx.find(r);
        if (it != xrow_idx.end()) return it->second;
        const uint32_t idx = (uint32_t)(xrows.size() / xcls);
        xrows.insert(xrows.end(), r.begin(), r.end());
        xrow_idx.emplace(r, idx);
        return idx;
    };

    // ---- EFT image (NEXT f4): forward in-arcs by π position, any K
    {
        std::vector<GOp> go(K);
        std::vector<GArc> ga;
        for (int p = 0; p < K; p++) {
            GOp &o = go[p];
            memset(&o, 0, sizeof o);
            o.fwd = d->fwd_ps[pi[p]];
            o.mem = d->mem_bytes ? d->mem_bytes[pi[p]] : 0;
            o.in_begin = (uint32_t)ga.size();
            for (int e : in_e[p]) ga.push_back(GArc{(uint32_t)pos[src[e]], xrow(e, false)});
            o.in_cnt = (uint32_t)(ga.size() - o.in_begin);
        }
        size_t o = sizeof(GOp) * K;
        g->g_off_arc = (uint32_t)o;
        o = (o + sizeof(GArc) * ga.size() + 7) & ~size_t(7);
        g->g_off_rows = (uint32_t)o;
        // rows are appended after the exact image is built (it may add rows)
        g->gimage.assign(o, 0);
        memcpy(g->gimage.data(), go.data(), sizeof(GOp) * K);
        if (!ga.empty()) memcpy(g->gimage.data() + g->g_off_arc, ga.data(), sizeof(GArc) * ga.size());
    }

    // ---- exact-schedule image (NEXT f1)
    if (2 * K <= kMaxExactNodes) {
        const int N = 2 * K;
        bool ok = true;
        std::vector<XNode> xn(N);
        std::vector<XPred> xp;
        std::vector<std::vector<int>> succ(N);
        for (int n = 0; n < N; n++) {
            const bool f = n < K;
            const int p = f ? n : n - K;
            XNode &x = xn[n];
            memset(&x, 0, sizeof x);
            x.dur = f ? d->fwd_ps[pi[p]] : d->bwd_ps[pi[p]];
            x.pos = (uint8_t)p;
            x.pred_begin = (uint16_t)xp.size();
            auto arc = [&](int q, uint32_t row) {
                if (row > 0xFFFF) ok = false;
                xp.push_back(XPred{(uint8_t)q, 0, (uint16_t)row});
                x.predmask |= 1ull << q;
                succ[q].push_back(n);
            };
            if (f) {
                for (int e : in_e[p]) arc(pos[src[e]], xrow(e, false));
            } else {
                arc(p, 0);                                      // own forward (R1)
                for (int e : out_e[p]) arc(K + pos[dst[e]], xrow(e, true));
            }
            const size_t np = xp.size() - x.pred_begin;
            if (np > 255 || xp.size() > 0xFFFF) ok = false;
            x.npred = (uint8_t)np;
        }
        // tail0 over the reverse of the topological order F_0..F_{K−1}, B_{K−1}..B_0
        for (int t = N - 1; t >= 0; t--) {
            const int n = t < K ? t : N - 1 - (t - K);
            uint64_t m = 0;
            for (int s2 : succ[n]) m = std::max(m, xn[s2].tail0);
            xn[n].tail0 = xn[n].dur + m;
        }
        if (ok) {
            size_t o = sizeof(XNode) * N;
            g->x_off_pred = (uint32_t)o;
            o = (o + sizeof(XPred) * xp.size() + 7) & ~size_t(7);
            g->x_off_rows = (uint32_t)o;
            o += 8 * xrows.size();
            g->x_off_cls = (uint32_t)o;
            o += 64;
            g->x_off_mem = (uint32_t)o;
            o += 8ull * K;
            g->x_off_orig = (uint32_t)o;
            o = (o + K + 15) & ~size_t(15);
            if (o <= (size_t)kMaxImageBytes) {
                g->ximage.assign(o, 0);
                memcpy(g->ximage.data(), xn.data(), sizeof(XNode) * N);
                if (!xp.empty()) memcpy(g->ximage.data() + g->x_off_pred, xp.data(), sizeof(XPred) * xp.size());
                memcpy(g->ximage.data() + g->x_off_rows, xrows.data(), 8 * xrows.size());
                memcpy(g->ximage.data() + g->x_off_cls, xc.data(), 64);
                for (int p = 0; p < K; p++) {
                    uint64_t m = d->mem_bytes ? d->mem_bytes[pi[p]] : 0;
                    memcpy(g->ximage.data() + g->x_off_mem + 8ull * p, &m, 8);
                    g->ximage[g->x_off_orig + p] = (uint8_t)pi[p];
                }
                g->xN = (uint32_t)N;
                g->xcls = (uint32_t)xcls;
                g->x_bytes = (uint32_t)o;
            }
        }
    }

    {   // EFT image: rows and class table
        size_t o = g->g_off_rows;
        g->gimage.resize(o + 8 * xrows.size());
        memcpy(g->gimage.data() + o, xrows.data(), 8 * xrows.size());
        o += 8 * xrows.size();
        g->g_off_cls = (uint32_t)o;
        g->gimage.resize((o + 64 + 15) & ~size_t(15), 0);
        memcpy(g->gimage.data() + o, xc.data(), 64);
        g->gcls = (uint32_t)xcls;
        g->g_bytes = (uint32_t)g->gimage.size();
    }

    // ---- device side
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t ce = cudaSetDevice(cuda_device);
    auto cuda_fail = [&](cudaError_t err) {
        set_error(std::string("CUDA: ") + cudaGetErrorString(err));
        cudaSetDevice(prev);
        return PP_E_CUDA;
    };
    if (ce != cudaSuccess) { delete g; return cuda_fail(ce); }
    cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, cuda_device);
    size_t scal = 64;   // u64 scalars
    if ((ce = cudaMalloc(&g->d_image, bytes)) != cudaSuccess ||
        (ce = cudaMalloc(&g->d_base, 3 * g->base_bytes)) != cudaSuccess ||
        (ce = cudaMalloc(&g->d_partials, sizeof(uint64_t) * 2 * kMaxGrid)) != cudaSuccess ||
        (ce = cudaMalloc(&g->d_ticket, sizeof(unsigned) * 8)) != cudaSuccess ||
        (ce = cudaMalloc(&g->d_scalars, sizeof(uint64_t) * scal)) != cudaSuccess) {
        pp_free_dfg(g);
        return cuda_fail(ce);
    }
    if ((ce = cudaMalloc(&g->d_gimage, g->g_bytes)) != cudaSuccess ||
        (ce = cudaMemcpy(g->d_gimage, g->gimage.data(), g->g_bytes, cudaMemcpyHostToDevice)) != cudaSuccess) {
        pp_free_dfg(g);
        return cuda_fail(ce);
    }
    if (g->x_bytes &&
        ((ce = cudaMalloc(&g->d_ximage, g->x_bytes)) != cudaSuccess ||
         (ce = cudaMalloc(&g->d_xwork, sizeof(unsigned long long) * 4)) != cudaSuccess ||
         (ce = cudaMemcpy(g->d_ximage, g->ximage.data(), g->x_bytes, cudaMemcpyHostToDevice)) != cudaSuccess)) {
        pp_free_dfg(g);
        return cuda_fail(ce);
    }
    g->d_winner = g->d_base + g->base_bytes;
    g->d_best_place = g->d_base + 2 * g->base_bytes;
    if ((ce = cudaMemcpy(g->d_image, g->image.data(), bytes, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (ce = cudaMemset(g->d_base, 0, 3 * g->base_bytes)) != cudaSuccess ||
        (ce = cudaMemset(g->d_ticket, 0, sizeof(unsigned) * 8)) != cudaSuccess ||
        (ce = cudaMemset(g->d_scalars, 0, sizeof(uint64_t) * scal)) != cudaSuccess) {
        pp_free_dfg(g);
        return cuda_fail(ce);
    }
    cudaSetDevice(prev);
    *out = g;
    return PP_OK;
}

}  // namespace pp

extern "C" void pp_free_dfg(pp_dfg *g) {
    if (!g) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(g->device);
    if (g->d_image) cudaFree(g->d_image);
    if (g->d_base) cudaFree(g->d_base);
    if (g->d_partials) cudaFree(g->d_partials);
    if (g->d_ticket) cudaFree(g->d_ticket);
    if (g->d_scalars) cudaFree(g->d_scalars);
    if (g->d_ximage) cudaFree(g->d_ximage);
    if (g->d_xwork) cudaFree(g->d_xwork);
    if (g->d_gimage) cudaFree(g->d_gimage);
    if (g->d_pipe) cudaFree(g->d_pipe);
    if (g->d_rgs) cudaFree(g->d_rgs);
    if (g->d_state) cudaFree(g->d_state);
    cudaSetDevice(prev);
    delete g;
}
