"""Independent brute-force checker for the oracle (pin K16).

It shares nothing with oracle/pp_oracle.c: a different formulation of the same
quantity.  The step makespan of a placement is the LONGEST PATH of an
augmented DAG over 2K nodes (forward node F_k, backward node B_k):

  * node weight = Δf(k) for F_k, Δb(k) for B_k;
  * data edge F_u → F_v for every DFG edge (u, v) with weight c_f(e) if u and v
    sit on different devices (the dependency constraint with
    Δ_e), and the reversed gradient edge B_v → B_u with c_b(e) (reading R1);
  * F_k → B_k for every op (a backward op never precedes its own forward);
  * device-order edges between consecutive ops of one device in the issue
    sequence F_π0..F_πK−1, B_πK−1..B_π0 (reading R2: in-order per-device issue,
    PAPER.md:465–476 non-overlap, PAPER.md:501 back-to-back).

The longest path is evaluated by memoised recursion over predecessors, not by
walking the issue sequence.  Exhaustive search enumerates placements with
itertools.product; Gray order is the textbook recursive reflected M-ary Gray
list (not the digit rule of O5).
"""
from __future__ import annotations

import functools
import heapq
import itertools
import sys


def kahn_by_id(K, ids, src, dst):
    indeg = [0] * K
    succ = [[] for _ in range(K)]
    for u, v in zip(src, dst):
        indeg[v] += 1
        succ[u].append(v)
    heap = [(ids[k], k) for k in range(K) if indeg[k] == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        _, k = heapq.heappop(heap)
        order.append(k)
        for v in succ[k]:
            indeg[v] -= 1
            if indeg[v] == 0:
                heapq.heappush(heap, (ids[v], v))
    if len(order) != K:
        raise ValueError("cycle")
    return order


def _cost(nbytes, bw, lat):
    return -(-nbytes * 10**12 // bw) + lat


def route_delays(hw, nbytes):
    """All-pairs delay of the cheapest route for a payload of `nbytes` on the
    hardware graph (PAPER.md:352 nodes N ∪ R and links L; Δ_e of PAPER.md:455–462
    summed over the route's links), by Floyd–Warshall over device and router
    nodes — a different algorithm from the oracle's Dijkstra.  Returns
    d[a][b] for devices a, b (None if unreachable)."""
    V = hw["num_devices"] + hw.get("num_routers", 0)
    INF = None
    d = [[0 if i == j else INF for j in range(V)] for i in range(V)]
    for a, b, bw, lat in zip(hw["link_a"], hw["link_b"], hw["link_bw_Bps"], hw["link_lat_ps"]):
        c = _cost(nbytes, bw, lat)
        for x, y in ((a, b), (b, a)):
            if d[x][y] is None or c < d[x][y]:
                d[x][y] = c
    for k in range(V):
        for i in range(V):
            if d[i][k] is None:
                continue
            for j in range(V):
                if d[k][j] is not None and (d[i][j] is None or d[i][k] + d[k][j] < d[i][j]):
                    d[i][j] = d[i][k] + d[k][j]
    nd = hw["num_devices"]
    return [row[:nd] for row in d[:nd]]


def longest_path_makespan(spec, M, placement):
    K = len(spec["fwd_ps"])
    ids = spec.get("op_id") or list(range(K))
    src, dst = spec["edge_src"], spec["edge_dst"]
    bf = spec["edge_fwd_bytes"]
    bb = spec.get("edge_bwd_bytes") or bf
    hw = spec.get("hw")
    if hw is None:
        bw, lat = spec["link_bw_Bps"], spec["link_lat_ps"]

        def cost(nbytes, a, b):
            return _cost(nbytes, bw, lat) if a != b else 0
    else:
        memo = {}

        def cost(nbytes, a, b):
            if nbytes not in memo:
                memo[nbytes] = route_delays(hw, nbytes)
            return memo[nbytes][a][b]
    order = kahn_by_id(K, ids, src, dst)
    seq = [("F", k) for k in order] + [("B", k) for k in reversed(order)]
    preds = {n: [] for n in seq}
    for e, (u, v) in enumerate(zip(src, dst)):
        a, b = placement[u], placement[v]
        preds[("F", v)].append((("F", u), cost(bf[e], a, b)))
        preds[("B", u)].append((("B", v), cost(bb[e], b, a)))
    for k in range(K):
        preds[("B", k)].append((("F", k), 0))
    last = {}
    for n in seq:
        dev = placement[n[1]]
        if dev in last:
            preds[n].append((last[dev], 0))
        last[dev] = n
    w = {("F", k): spec["fwd_ps"][k] for k in range(K)}
    w.update({("B", k): spec["bwd_ps"][k] for k in range(K)})
    sys.setrecursionlimit(max(10000, 8 * K + 100))

    @functools.lru_cache(maxsize=None)
    def finish(n):
        s = 0
        for p, c in preds[n]:
            s = max(s, finish(p) + c)
        return s + w[n]

    mk = max(finish(n) for n in seq)
    cap = (hw or spec).get("dev_mem_cap_bytes") or 0
    if cap:
        mem = spec.get("mem_bytes") or [0] * K
        for m in range(M):
            if sum(mem[k] for k in range(K) if placement[k] == m) > cap:
                return (1 << 64) - 1
    return mk


def exact_makespan(spec, M, placement):
    """Makespan-optimal schedule of a fixed placement (NEXT f1), by the
    disjunctive-graph formulation: choose an order of the nodes on every
    device (all permutations, per device), add the consecutive-order arcs to
    the precedence arcs of the augmented DAG; if the result is acyclic its
    longest path is that choice's makespan.  Minimum over every choice.  A
    different formulation from the oracle's enumeration of linear extensions."""
    K = len(spec["fwd_ps"])
    src, dst = spec["edge_src"], spec["edge_dst"]
    bf = spec["edge_fwd_bytes"]
    bb = spec.get("edge_bwd_bytes") or bf
    hw = spec.get("hw")
    cap = (hw or spec).get("dev_mem_cap_bytes") or 0
    if cap:
        mem = spec.get("mem_bytes") or [0] * K
        for m in range(M):
            if sum(mem[k] for k in range(K) if placement[k] == m) > cap:
                return (1 << 64) - 1
    if hw is None:
        bw, lat = spec["link_bw_Bps"], spec["link_lat_ps"]

        def cost(nbytes, a, b):
            return _cost(nbytes, bw, lat) if a != b else 0
    else:
        def cost(nbytes, a, b):
            return route_delays(hw, nbytes)[a][b]
    nodes = [("F", k) for k in range(K)] + [("B", k) for k in range(K)]
    w = {("F", k): spec["fwd_ps"][k] for k in range(K)}
    w.update({("B", k): spec["bwd_ps"][k] for k in range(K)})
    arcs = []
    for e, (u, v) in enumerate(zip(src, dst)):
        a, b = placement[u], placement[v]
        arcs.append((("F", u), ("F", v), cost(bf[e], a, b)))
        arcs.append((("B", v), ("B", u), cost(bb[e], b, a)))
    arcs += [(("F", k), ("B", k), 0) for k in range(K)]
    per_dev = [[n for n in nodes if placement[n[1]] == m] for m in range(M)]
    best = None
    for orders in itertools.product(*[itertools.permutations(g) for g in per_dev]):
        extra = [(o[i], o[i + 1], 0) for o in orders for i in range(len(o) - 1)]
        preds = {n: [] for n in nodes}
        for a, b, c in arcs + extra:
            preds[b].append((a, c))
        fin, state, ok = {}, {}, [True]

        def visit(n):
            if state.get(n) == 2:
                return fin[n]
            if state.get(n) == 1:
                ok[0] = False
                return 0
            state[n] = 1
            s = 0
            for p, c in preds[n]:
                s = max(s, visit(p) + c)
            state[n] = 2
            fin[n] = s + w[n]
            return fin[n]

        mk = max(visit(n) for n in nodes)
        if ok[0] and (best is None or mk < best):
            best = mk
    return best


def reflected_gray(M, K):
    """Textbook recursive reflected M-ary Gray list; tuple index j = digit j
    (digit 0 changes fastest)."""
    L = [(a,) for a in range(M)]
    for _ in range(1, K):
        nxt = []
        for a in range(M):
            block = L if a % 2 == 0 else list(reversed(L))
            nxt.extend(t + (a,) for t in block)
        L = nxt
    return L


def exhaustive(spec, M):
    """(best makespan, number of optimal placements, all optima) by brute force."""
    K = len(spec["fwd_ps"])
    best, opt = None, []
    for pl in itertools.product(range(M), repeat=K):
        mk = longest_path_makespan(spec, M, pl)
        if best is None or mk < best:
            best, opt = mk, [pl]
        elif mk == best:
            opt.append(pl)
    return best, opt


def gray_first_index(spec, M, best):
    """Index, in Gray order over π positions, of the first optimal placement."""
    K = len(spec["fwd_ps"])
    ids = spec.get("op_id") or list(range(K))
    order = kahn_by_id(K, ids, spec["edge_src"], spec["edge_dst"])
    for i, g in enumerate(reflected_gray(M, K)):
        pl = [0] * K
        for j, k in enumerate(order):
            pl[k] = g[j]
        if longest_path_makespan(spec, M, pl) == best:
            return i, pl
    return None, None


def pipeline_makespan(spec, M, cuts, m):
    """GPipe makespan (NEXT f3, reading R26) as the longest path of an explicit
    task graph: tasks F(s,j) and B(s,j) with their micro-batch times; arcs for
    each device's task order F(s,0..m−1), B(s,m−1..0) and for the stage-to-
    stage transfers of every micro-batch.  A different formulation from the
    oracle's row recurrences."""
    K = len(spec["fwd_ps"])
    ids = spec.get("op_id") or list(range(K))
    order = kahn_by_id(K, ids, spec["edge_src"], spec["edge_dst"])
    bounds = [0] + list(cuts) + [K]
    stage = {}
    for s in range(M):
        for p in range(bounds[s], bounds[s + 1]):
            stage[order[p]] = s
    cap = spec.get("dev_mem_cap_bytes") or 0
    if cap:
        mem = spec.get("mem_bytes") or [0] * K
        for s in range(M):
            if sum(mem[k] for k in range(K) if stage[k] == s) > cap:
                return (1 << 64) - 1
    tf = [-(-sum(spec["fwd_ps"][k] for k in range(K) if stage[k] == s) // m) for s in range(M)]
    tb = [-(-sum(spec["bwd_ps"][k] for k in range(K) if stage[k] == s) // m) for s in range(M)]
    bf = spec["edge_fwd_bytes"]
    bb = spec.get("edge_bwd_bytes") or bf
    bw, lat = spec["link_bw_Bps"], spec["link_lat_ps"]
    link = {}
    for e, (u, v) in enumerate(zip(spec["edge_src"], spec["edge_dst"])):
        a, b = stage[u], stage[v]
        if a != b:
            x = link.setdefault((a, b), [0, 0])
            x[0] += bf[e]
            x[1] += bb[e]
    preds = {}
    for s in range(M):
        seq = [("F", s, j) for j in range(m)] + [("B", s, j) for j in reversed(range(m))]
        for i, t in enumerate(seq):
            preds[t] = [(seq[i - 1], 0)] if i else []
    for (a, b), (df, db) in link.items():
        for j in range(m):
            preds[("F", b, j)].append((("F", a, j), -(-df * 10**12 // (m * bw)) + lat))
            preds[("B", a, j)].append((("B", b, j), -(-db * 10**12 // (m * bw)) + lat))
    dur = {("F", s, j): tf[s] for s in range(M) for j in range(m)}
    dur.update({("B", s, j): tb[s] for s in range(M) for j in range(m)})
    memo = {}

    def fin(t):
        if t not in memo:
            memo[t] = max([fin(p) + c for p, c in preds[t]] or [0]) + dur[t]
        return memo[t]

    return max(fin(("B", s, 0)) for s in range(M))
