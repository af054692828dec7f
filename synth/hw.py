"""Seeded synthetic hardware graphs ("a set of
compute nodes N and router nodes R connected through a set of physical links
L", bandwidth B(l); Table 2).  Node ids: devices
0..num_devices−1, routers num_devices.. .  Each function returns the dict
pp.Dfg / oracle.Dfg take as spec["hw"].  No arithmetic of the method here.

Bandwidths in B/s, latencies in ps.  The figures are round numbers of the
interconnect class each topology is named after (NVLink-era per-link rates),
not measurements.
"""
from __future__ import annotations

import numpy as np

NVLINK_BW = 25_000_000_000       # one NVLink 2 link, B/s per direction (V100 era)
NVLINK_LAT = 1_000_000           # 1 µs
IB_BW = 12_500_000_000           # 100 Gb/s InfiniBand
IB_LAT = 5_000_000               # 5 µs


def _hw(nd, nr, links, cap=0):
    a, b, bw, lat = zip(*links)
    return {"num_devices": nd, "num_routers": nr, "link_a": list(a), "link_b": list(b),
            "link_bw_Bps": list(bw), "link_lat_ps": list(lat), "dev_mem_cap_bytes": cap}


def full_mesh(nd, bw=NVLINK_BW, lat=NVLINK_LAT, cap=0):
    """A direct link between every device pair: the uniform-link model."""
    return _hw(nd, 0, [(i, j, bw, lat) for i in range(nd) for j in range(i + 1, nd)], cap)


def switch(nd, bw=NVLINK_BW, lat=NVLINK_LAT, cap=0):
    """Every device on one router (an NVSwitch / PCIe switch): two hops per transfer."""
    return _hw(nd, 1, [(i, nd, bw, lat) for i in range(nd)], cap)


def ring(nd, bw=NVLINK_BW, lat=NVLINK_LAT, cap=0):
    return _hw(nd, 0, [(i, (i + 1) % nd, bw, lat) for i in range(nd)] if nd > 2 else [(0, 1, bw, lat)], cap)


def hybrid_cube_mesh(bw=NVLINK_BW, lat=NVLINK_LAT, cap=0):
    """8 devices after the DGX-1 hybrid cube-mesh: two fully connected quads
    {0..3}, {4..7} plus the links i – i+4; pairs (0,3), (1,2), (4,7), (5,6) and
    the cross links carry a doubled link (2·bw).  Pairs without a direct link
    route over two hops."""
    links = []
    for q in (0, 4):
        for i in range(4):
            for j in range(i + 1, 4):
                dbl = (i, j) in ((0, 3), (1, 2))
                links.append((q + i, q + j, 2 * bw if dbl else bw, lat))
    links += [(i, i + 4, 2 * bw, lat) for i in range(4)]
    return _hw(8, 0, links, cap)


def two_nodes(per_node=4, bw=NVLINK_BW, lat=NVLINK_LAT, ib_bw=IB_BW, ib_lat=IB_LAT, cap=0):
    """Two nodes of `per_node` devices, each node behind its own switch, the
    switches joined by one network link."""
    nd = 2 * per_node
    r0, r1 = nd, nd + 1
    links = [(i, r0 if i < per_node else r1, bw, lat) for i in range(nd)]
    links.append((r0, r1, ib_bw, ib_lat))
    return _hw(nd, 2, links, cap)


def random_hw(seed, nd, nr=2, extra_links=4, cap=0):
    """A random connected graph: a random spanning tree over devices and
    routers plus `extra_links` random links; bandwidths 1–64 GB/s, latencies
    0–5 µs."""
    rng = np.random.default_rng(seed)
    V = nd + nr
    order = rng.permutation(V)
    links = []
    for i in range(1, V):
        links.append((int(order[i]), int(order[rng.integers(0, i)])))
    for _ in range(extra_links):
        a, b = rng.choice(V, 2, replace=False)
        links.append((int(a), int(b)))
    return _hw(nd, nr, [(a, b, int(rng.integers(1, 65)) * 1_000_000_000, int(rng.integers(0, 5_000_001)))
                        for a, b in links], cap)


TOPOLOGIES = {
    "full_mesh": full_mesh,
    "switch": switch,
    "ring": ring,
}
