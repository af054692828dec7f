"""Synthetic training DFGs shaped like the paper's workloads.

Op times follow the analytic recipe of PAPER.md:511 (§6 case study: FLOPs over
the advertised compute rate; bytes over bandwidth plus latency), made exact in
integer picoseconds as reading R20 states:

  matmul/conv op   Δf = ⌈FLOPs·10^12 / F_peak⌉ + ℓ,   Δb = 2·(Δf − ℓ) + ℓ
  elementwise op   Δf = ⌈2·bytes·10^12 / HBM⌉ + ℓ,     Δb = Δf

Edge bytes D(e) are the producer's output activation ("the amount
of total output activation"); gradient bytes default to the same (R1).
Layer shapes: Inception-V3 from the public torchvision layer table; GNMT from
PAPER.md:230 (4+4 LSTM × 1024); BigLSTM from PAPER.md:232 (emb 1024, 2 × LSTM
8192 with 1024 projection).  Everything else (batch, sequence chunking, vocab,
hardware profile) is synthetic and stated in DESIGN.md §Inputs.

A DFG spec is a plain dict of lists (descriptor order) consumed by both the
oracle and the CUDA library.
"""
from __future__ import annotations

import random

# hardware profiles used only to SHAPE synthetic costs (not part of parity)
PAPER_PROFILE = dict(flops=15_700_000_000_000, hbm=900_000_000_000, launch_ps=5_000_000,
                     link_bw=150_000_000_000, link_lat_ps=2_000_000)   # V100 / DGX-1 class
B200_PROFILE = dict(flops=80_000_000_000_000, hbm=7_700_000_000_000, launch_ps=3_000_000,
                    link_bw=900_000_000_000, link_lat_ps=1_000_000)


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


class _Builder:
    def __init__(self, profile, batch, dtype_bytes=4):
        self.p = profile
        self.B = batch
        self.db = dtype_bytes
        self.names, self.fwd, self.bwd, self.mem, self.par, self.ids = [], [], [], [], [], []
        self.src, self.dst, self.byt = [], [], []
        self.out_bytes = []

    def _add(self, name, fwd, bwd, out_bytes, params=0):
        self.names.append(name)
        self.fwd.append(int(fwd)); self.bwd.append(int(bwd))
        self.mem.append(int(out_bytes)); self.par.append(int(params))
        self.out_bytes.append(int(out_bytes))
        self.ids.append(len(self.ids))
        return len(self.names) - 1

    def compute(self, name, flops, out_elems, params=0, inputs=()):
        l = self.p["launch_ps"]
        core = _ceil_div(int(flops) * 10**12, self.p["flops"])
        k = self._add(name, core + l, 2 * core + l, out_elems * self.db, params * self.db)
        for u in inputs:
            self.edge(u, k)
        return k

    def elementwise(self, name, in_elems, out_elems, inputs=(), params=0):
        l = self.p["launch_ps"]
        core = _ceil_div(2 * int(in_elems) * self.db * 10**12, self.p["hbm"])
        k = self._add(name, core + l, core + l, out_elems * self.db, params * self.db)
        for u in inputs:
            self.edge(u, k)
        return k

    def edge(self, u, v, nbytes=None):
        self.src.append(u); self.dst.append(v)
        self.byt.append(int(self.out_bytes[u] if nbytes is None else nbytes))

    def spec(self, name, **extra):
        d = dict(name=name, names=self.names, op_id=self.ids, fwd_ps=self.fwd, bwd_ps=self.bwd,
                 mem_bytes=self.mem, param_bytes=self.par, edge_src=self.src, edge_dst=self.dst,
                 edge_fwd_bytes=self.byt, edge_bwd_bytes=None,
                 link_bw_Bps=self.p["link_bw"], link_lat_ps=self.p["link_lat_ps"],
                 dev_mem_cap_bytes=0)
        d.update(extra)
        return d


# --------------------------------------------------------------- toy-12
def toy12():
    """12 ops, 13 edges; µs times, 1 MB = 10^6 B,
    BW 10^11 B/s, L = 2 µs."""
    us = 1_000_000
    names = ["input", "conv_a", "conv_b1", "conv_b2", "conv_c1", "conv_c2", "conv_c3",
             "pool_d", "conv_d", "concat", "fc", "loss"]
    fwd = [10, 80, 60, 60, 40, 40, 40, 20, 30, 10, 50, 10]
    bwd = [0, 160, 120, 120, 80, 80, 80, 20, 60, 10, 100, 10]
    MB = 10**6
    edges = [(0, 1, 2 * MB), (1, 2, MB), (2, 3, MB), (1, 4, MB), (4, 5, MB), (5, 6, MB),
             (1, 7, MB), (7, 8, MB), (3, 9, MB), (6, 9, MB), (8, 9, MB), (9, 10, 2 * MB),
             (10, 11, 4096)]
    return dict(name="toy12", names=names, op_id=list(range(12)),
                fwd_ps=[x * us for x in fwd], bwd_ps=[x * us for x in bwd],
                mem_bytes=None, param_bytes=[0, 10**6, 10**6, 10**6, 10**6, 10**6, 10**6, 0,
                                             10**6, 0, 4 * 10**6, 0],
                edge_src=[e[0] for e in edges], edge_dst=[e[1] for e in edges],
                edge_fwd_bytes=[e[2] for e in edges], edge_bwd_bytes=None,
                link_bw_Bps=10**11, link_lat_ps=2 * us, dev_mem_cap_bytes=0)


# ---------------------------------------------------------- Inception-V3
def inception_v3(batch=64, profile=PAPER_PROFILE):
    """Inception-V3-shaped DFG (torchvision layer table, 299×299 input),
    conv units expanded to conv→bn→relu (TF-op granularity),
    aux head, single sink (total loss)."""
    b = _Builder(profile, batch)
    B = batch

    def conv(tag, x, cin, cout, kh, kw, hout, wout):
        flops = 2 * B * hout * wout * cout * cin * kh * kw
        n = B * hout * wout * cout
        c = b.compute(f"{tag}/conv", flops, n, params=kh * kw * cin * cout, inputs=[x])
        bn = b.elementwise(f"{tag}/bn", n, n, inputs=[c], params=2 * cout)
        return b.elementwise(f"{tag}/relu", n, n, inputs=[bn])

    def pool(tag, x, c, hin, win, hout, wout):
        return b.elementwise(tag, B * hin * win * c, B * hout * wout * c, inputs=[x])

    def concat(tag, xs, c, h, w):
        n = B * h * w * c
        return b.elementwise(tag, n, n, inputs=xs)

    x = b.elementwise("input", B * 299 * 299 * 3, B * 299 * 299 * 3)
    x = conv("Conv2d_1a", x, 3, 32, 3, 3, 149, 149)
    x = conv("Conv2d_2a", x, 32, 32, 3, 3, 147, 147)
    x = conv("Conv2d_2b", x, 32, 64, 3, 3, 147, 147)
    x = pool("maxpool1", x, 64, 147, 147, 73, 73)
    x = conv("Conv2d_3b", x, 64, 80, 1, 1, 73, 73)
    x = conv("Conv2d_4a", x, 80, 192, 3, 3, 71, 71)
    x = pool("maxpool2", x, 192, 71, 71, 35, 35)

    def block_a(tag, x, cin, pf):
        s = 35
        b1 = conv(f"{tag}/b1x1", x, cin, 64, 1, 1, s, s)
        b5 = conv(f"{tag}/b5x5_1", x, cin, 48, 1, 1, s, s)
        b5 = conv(f"{tag}/b5x5_2", b5, 48, 64, 5, 5, s, s)
        b3 = conv(f"{tag}/b3dbl_1", x, cin, 64, 1, 1, s, s)
        b3 = conv(f"{tag}/b3dbl_2", b3, 64, 96, 3, 3, s, s)
        b3 = conv(f"{tag}/b3dbl_3", b3, 96, 96, 3, 3, s, s)
        bp = pool(f"{tag}/avgpool", x, cin, s, s, s, s)
        bp = conv(f"{tag}/bpool", bp, cin, pf, 1, 1, s, s)
        return concat(f"{tag}/concat", [b1, b5, b3, bp], 224 + pf, s, s), 224 + pf

    x, c = block_a("Mixed_5b", x, 192, 32)
    x, c = block_a("Mixed_5c", x, c, 64)
    x, c = block_a("Mixed_5d", x, c, 64)

    # Mixed_6a (reduction)
    b3 = conv("Mixed_6a/b3x3", x, c, 384, 3, 3, 17, 17)
    bd = conv("Mixed_6a/b3dbl_1", x, c, 64, 1, 1, 35, 35)
    bd = conv("Mixed_6a/b3dbl_2", bd, 64, 96, 3, 3, 35, 35)
    bd = conv("Mixed_6a/b3dbl_3", bd, 96, 96, 3, 3, 17, 17)
    bp = pool("Mixed_6a/maxpool", x, c, 35, 35, 17, 17)
    x = concat("Mixed_6a/concat", [b3, bd, bp], 768, 17, 17)
    c = 768

    def block_c(tag, x, c7):
        s = 17
        b1 = conv(f"{tag}/b1x1", x, 768, 192, 1, 1, s, s)
        b7 = conv(f"{tag}/b7_1", x, 768, c7, 1, 1, s, s)
        b7 = conv(f"{tag}/b7_2", b7, c7, c7, 1, 7, s, s)
        b7 = conv(f"{tag}/b7_3", b7, c7, 192, 7, 1, s, s)
        bd = conv(f"{tag}/b7dbl_1", x, 768, c7, 1, 1, s, s)
        bd = conv(f"{tag}/b7dbl_2", bd, c7, c7, 7, 1, s, s)
        bd = conv(f"{tag}/b7dbl_3", bd, c7, c7, 1, 7, s, s)
        bd = conv(f"{tag}/b7dbl_4", bd, c7, c7, 7, 1, s, s)
        bd = conv(f"{tag}/b7dbl_5", bd, c7, 192, 1, 7, s, s)
        bp = pool(f"{tag}/avgpool", x, 768, s, s, s, s)
        bp = conv(f"{tag}/bpool", bp, 768, 192, 1, 1, s, s)
        return concat(f"{tag}/concat", [b1, b7, bd, bp], 768, s, s)

    x = block_c("Mixed_6b", x, 128)
    x = block_c("Mixed_6c", x, 160)
    x = block_c("Mixed_6d", x, 160)
    x = block_c("Mixed_6e", x, 192)

    # aux head on Mixed_6e
    a = pool("Aux/avgpool", x, 768, 17, 17, 5, 5)
    a = conv("Aux/conv0", a, 768, 128, 1, 1, 5, 5)
    a = conv("Aux/conv1", a, 128, 768, 5, 5, 1, 1)
    a = b.compute("Aux/fc", 2 * B * 768 * 1000, B * 1000, params=768 * 1000, inputs=[a])
    aux_loss = b.elementwise("Aux/loss", B * 1000, B, inputs=[a])

    # Mixed_7a (reduction)
    b3 = conv("Mixed_7a/b3_1", x, 768, 192, 1, 1, 17, 17)
    b3 = conv("Mixed_7a/b3_2", b3, 192, 320, 3, 3, 8, 8)
    b7 = conv("Mixed_7a/b7_1", x, 768, 192, 1, 1, 17, 17)
    b7 = conv("Mixed_7a/b7_2", b7, 192, 192, 1, 7, 17, 17)
    b7 = conv("Mixed_7a/b7_3", b7, 192, 192, 7, 1, 17, 17)
    b7 = conv("Mixed_7a/b7_4", b7, 192, 192, 3, 3, 8, 8)
    bp = pool("Mixed_7a/maxpool", x, 768, 17, 17, 8, 8)
    x = concat("Mixed_7a/concat", [b3, b7, bp], 1280, 8, 8)
    c = 1280

    def block_e(tag, x, cin):
        s = 8
        b1 = conv(f"{tag}/b1x1", x, cin, 320, 1, 1, s, s)
        b3 = conv(f"{tag}/b3_1", x, cin, 384, 1, 1, s, s)
        b3a = conv(f"{tag}/b3_2a", b3, 384, 384, 1, 3, s, s)
        b3b = conv(f"{tag}/b3_2b", b3, 384, 384, 3, 1, s, s)
        b3 = concat(f"{tag}/b3_concat", [b3a, b3b], 768, s, s)
        bd = conv(f"{tag}/b3dbl_1", x, cin, 448, 1, 1, s, s)
        bd = conv(f"{tag}/b3dbl_2", bd, 448, 384, 3, 3, s, s)
        bda = conv(f"{tag}/b3dbl_3a", bd, 384, 384, 1, 3, s, s)
        bdb = conv(f"{tag}/b3dbl_3b", bd, 384, 384, 3, 1, s, s)
        bd = concat(f"{tag}/b3dbl_concat", [bda, bdb], 768, s, s)
        bp = pool(f"{tag}/avgpool", x, cin, s, s, s, s)
        bp = conv(f"{tag}/bpool", bp, cin, 192, 1, 1, s, s)
        return concat(f"{tag}/concat", [b1, b3, bd, bp], 2048, s, s)

    x = block_e("Mixed_7b", x, 1280)
    x = block_e("Mixed_7c", x, 2048)
    x = pool("avgpool", x, 2048, 8, 8, 1, 1)
    x = b.compute("fc", 2 * B * 2048 * 1000, B * 1000, params=2048 * 1000, inputs=[x])
    loss = b.elementwise("loss", B * 1000, B, inputs=[x])
    b.elementwise("total_loss", 2 * B, 1, inputs=[loss, aux_loss])
    return b.spec("inception_v3", batch=batch)


# ------------------------------------------------------------------ GNMT
def gnmt(batch=128, chunks=18, steps_per_chunk=3, hidden=1024, vocab=32000, profile=PAPER_PROFILE):
    """GNMT-shaped: 4 encoder + 4 decoder LSTM layers × `chunks` time chunks
    (PAPER.md:230), per-chunk attention over all encoder outputs and
    projection, a chained loss.  Ops numbered time-major (chunk by chunk).

    The embedding lookup of a chunk's tokens is part of its layer-0 LSTM op
    (cost and parameters), which reads the chunk's token slice of the input
    directly: a separate embedding op shared by every chunk would be a
    18-way fan-out whose backward waits for all 18 chunks — a data input has
    no gradient, and it kept 18 extra finish times live (W 38 → 22; DESIGN.md
    §4).  The attention's 18-way fan-in (enc_concat) and fan-out (every
    decoder chunk attends to all encoder outputs) is the model's, so W = 22
    remains."""
    b = _Builder(profile, batch)
    B, H, T = batch, hidden, steps_per_chunk
    lstm_flops = 2 * B * 4 * H * (H + H) * T
    act = B * T * H
    state = 2 * B * H
    emb_flops = 2 * B * T * H          # the lookup's gather (per chunk)
    enc = [[None] * chunks for _ in range(4)]
    for t in range(chunks):
        for l in range(4):
            ins = [] if l == 0 else [enc[l - 1][t]]
            k = b.compute(f"enc{l}/t{t}", lstm_flops + (emb_flops if l == 0 else 0), act,
                          params=((8 * H * H) if t == 0 else 0) + ((vocab * H) if (t == 0 and l == 0) else 0),
                          inputs=ins)
            if t > 0:
                b.edge(enc[l][t - 1], k, nbytes=state * b.db)
            enc[l][t] = k
    enc_cat = b.elementwise("enc_concat", act * chunks, act * chunks, inputs=[enc[3][t] for t in range(chunks)])
    dec = [[None] * chunks for _ in range(4)]
    loss_prev = None
    for t in range(chunks):
        for l in range(4):
            ins = [] if l == 0 else [dec[l - 1][t]]
            k = b.compute(f"dec{l}/t{t}", (lstm_flops + emb_flops) if l == 0 else 2 * B * 4 * H * 3 * H * T, act,
                          params=((8 * H * H) if t == 0 else 0) + ((vocab * H) if (t == 0 and l == 0) else 0),
                          inputs=ins)
            if t > 0:
                b.edge(dec[l][t - 1], k, nbytes=state * b.db)
            if l >= 1:
                b.edge(attn, k)
            dec[l][t] = k
            if l == 0:
                attn = b.compute(f"attn/t{t}", 2 * B * T * H * T * chunks * 2, act,
                                 params=(2 * H * H) if t == 0 else 0, inputs=[k, enc_cat])
        proj = b.compute(f"proj/t{t}", 2 * B * T * H * vocab, B * T * vocab,
                         params=(H * vocab) if t == 0 else 0, inputs=[dec[3][t]])
        ins = [proj] + ([loss_prev] if loss_prev is not None else [])
        loss_prev = b.elementwise(f"loss/t{t}", B * T * vocab, B * T, inputs=[proj])
        if len(ins) > 1:
            b.edge(ins[1], loss_prev, nbytes=4 * b.db)
    return b.spec("gnmt", batch=batch)


# --------------------------------------------------------------- BigLSTM
def biglstm(batch=128, chunks=30, steps_per_chunk=1, hidden=8192, proj=1024, emb=1024,
            sampled_softmax=8192, profile=PAPER_PROFILE):
    """BigLSTM-shaped: embedding 1024 → 2 × LSTM 8192 with 1024 projection →
    (sampled) softmax; time-major chunks; chained loss.

    Each chunk's embedding lookup reads its own token slice of the input (a
    source op): one input op feeding all 30 chunks would have no gradient to
    compute yet a backward waiting on all 30 chunks, keeping 30 finish times
    live (W 32 → 3)."""
    b = _Builder(profile, batch)
    B, H, P, T = batch, hidden, proj, steps_per_chunk
    l1 = [None] * chunks
    l2 = [None] * chunks
    loss_prev = None
    lstm_flops = (2 * B * 4 * H * (emb + P) + 2 * B * H * P) * T
    for t in range(chunks):
        e = b.elementwise(f"emb/t{t}", B * T * emb, B * T * emb, inputs=[],
                          params=(800_000 * emb) if t == 0 else 0)
        k1 = b.compute(f"lstm1/t{t}", lstm_flops, B * T * P,
                       params=(4 * H * (emb + P) + H * P) if t == 0 else 0, inputs=[e])
        if t > 0:
            b.edge(l1[t - 1], k1, nbytes=B * (H + P) * b.db)
        l1[t] = k1
        k2 = b.compute(f"lstm2/t{t}", lstm_flops, B * T * P,
                       params=(4 * H * 2 * P + H * P) if t == 0 else 0, inputs=[k1])
        if t > 0:
            b.edge(l2[t - 1], k2, nbytes=B * (H + P) * b.db)
        l2[t] = k2
        sm = b.compute(f"softmax/t{t}", 2 * B * T * P * sampled_softmax, B * T * sampled_softmax,
                       params=0, inputs=[k2])
        ls = b.elementwise(f"loss/t{t}", B * T * sampled_softmax, B * T, inputs=[sm])
        if loss_prev is not None:
            b.edge(loss_prev, ls, nbytes=4 * b.db)
        loss_prev = ls
    return b.spec("biglstm", batch=batch)


# ------------------------------------------------------- small fixtures
def _plain(name, fwd, bwd, edges, bw=10**12, lat=0, bwd_bytes=None, ids=None):
    return dict(name=name, names=[f"v{i}" for i in range(len(fwd))],
                op_id=ids if ids is not None else list(range(len(fwd))),
                fwd_ps=list(fwd), bwd_ps=list(bwd), mem_bytes=None, param_bytes=None,
                edge_src=[e[0] for e in edges], edge_dst=[e[1] for e in edges],
                edge_fwd_bytes=[e[2] for e in edges], edge_bwd_bytes=bwd_bytes,
                link_bw_Bps=bw, link_lat_ps=lat, dev_mem_cap_bytes=0)


def diamond(fwd=(2, 8, 8, 2), bwd=(0, 0, 0, 0), fwd_bytes=1, bwd_bytes=0, bw=10**12, lat=0):
    """SPEC.md:159–160 diamond 0→{1,2}→3.  With bw=10^12 B/s one byte costs 1 ps."""
    e = [(0, 1, fwd_bytes), (0, 2, fwd_bytes), (1, 3, fwd_bytes), (2, 3, fwd_bytes)]
    return _plain("diamond", fwd, bwd, e, bw, lat,
                  bwd_bytes=None if bwd_bytes is None else [bwd_bytes] * 4)


def chain(K, fwd, bwd, nbytes, bw=10**12, lat=0):
    e = [(k, k + 1, nbytes) for k in range(K - 1)]
    return _plain("chain", [fwd] * K if isinstance(fwd, int) else fwd,
                  [bwd] * K if isinstance(bwd, int) else bwd, e, bw, lat)


def star(leaves, d0, d, nbytes=0, bw=10**12, lat=0):
    e = [(0, k, nbytes) for k in range(1, leaves + 1)]
    return _plain("star", [d0] + [d] * leaves, [0] * (leaves + 1), e, bw, lat)


def independent(K, fwd, bwd):
    return _plain("independent", [fwd] * K, [bwd] * K, [])


def random_dag(seed, K, avg_deg=1.5, max_in=4, max_cost=1000, max_bytes=2000, bw=10**12,
               lat_max=50, zero_frac=0.05, shuffle_ids=True, param=False, window=None):
    """Seeded random DAG: edges only from lower to higher creation index, ids
    shuffled so π is not the identity; parallel edges allowed.
    `window` bounds how far back a producer may be (None = anywhere), which
    bounds the number of simultaneously live values like a real DFG."""
    rng = random.Random(seed)
    fwd = [0 if rng.random() < zero_frac else rng.randint(1, max_cost) for _ in range(K)]
    bwd = [0 if rng.random() < zero_frac else rng.randint(1, 2 * max_cost) for _ in range(K)]
    edges = []
    for v in range(1, K):
        nin = min(max_in, v, max(0, int(rng.expovariate(1.0 / avg_deg) + 0.5)))
        for _ in range(nin):
            lo = 0 if window is None else max(0, v - window)
            u = rng.randrange(lo, v) if rng.random() < 0.5 else max(0, v - 1 - rng.randrange(min(v, 4)))
            edges.append((u, v, rng.randint(0, max_bytes)))
    if window is not None:
        # like a training DFG, let only the last op be a sink: a sink's forward
        # finish time stays live until its own backward step
        has_out = set(u for u, _, _ in edges)
        for v in range(K - 1):
            if v not in has_out:
                edges.append((v, rng.randint(v + 1, min(K - 1, v + window)), rng.randint(0, max_bytes)))
    ids = list(range(K))
    if shuffle_ids and window is None:
        ids = rng.sample(range(10 * K), K)
    elif shuffle_ids:
        ids = sorted(rng.sample(range(10 * K), K))   # keep creation order = π (locality)
    bwd_bytes = [rng.randint(0, max_bytes) for _ in edges] if rng.random() < 0.5 else None
    d = _plain(f"random{seed}", fwd, bwd, edges, bw, rng.randint(0, lat_max), bwd_bytes=bwd_bytes,
               ids=ids)
    if param:
        d["param_bytes"] = [rng.randint(0, 10**6) for _ in range(K)]
        d["mem_bytes"] = [rng.randint(0, 1000) for _ in range(K)]
    return d
