"""Synthetic epochs-vs-global-batch curves and projection scenarios.

Curve shapes follow PAPER.md:304 (§5, Fig. 4 narrative): Inception-V3 epochs
4 → 7 once G > 2048 and 23 at G = 16384; BigLSTM 3.2× epochs from 16 to 32
GPUs; GNMT flat-ish then rapid growth beyond 64 GPUs.  Values are integer
µ-epochs (reading R12).  Knots beyond the paper-anchored points are synthetic
(DESIGN.md §Inputs).  Nothing here computes a projection.
"""
from __future__ import annotations

U = 10**9  # 1 ms in ps — the unit of the K10–K12 fixtures


def _knots(B, values):
    return [B * 2**k for k in range(len(values))], list(values)


def toy12_scenario(t1_ps, grad_bytes=40_000_000, ar_mode=0, ar_on=True):
    """B = 32, 16 knots G = 32·2^k, E = 10^7 µep flat
    for k ≤ 4 then ×1.6 per doubling (floor); D = 2^20."""
    vals = []
    e = 10**7
    for k in range(16):
        if k > 4:
            e = e * 16 // 10
        vals.append(e)
    G, E = _knots(32, vals)
    return dict(dataset_items=2**20, mini_batch=32, knot_G=G, knot_uepochs=E,
                grad_bytes=grad_bytes, t1_ps=t1_ps,
                bw_intra_Bps=150_000_000_000 if ar_on else 0, lat_intra_ps=2_000_000,
                bw_inter_Bps=50_000_000_000 if ar_on else 0, lat_inter_ps=5_000_000,
                node_size=8, ar_mode=ar_mode)


def _grow(head, factor_num, factor_den, n=16):
    vals = list(head)
    while len(vals) < n:
        vals.append(vals[-1] * factor_num // factor_den)
    return vals


SWEEP_CURVES = {
    # SURVEY.md §8(d) config 5 (k = 0..15 → G = B·2^k)
    "inception_v3": dict(B=64, D=1_281_167, vals=_grow([4 * 10**6] * 6 + [7 * 10**6, 12 * 10**6, 23 * 10**6], 2, 1)),
    "gnmt": dict(B=128, D=4_500_000, vals=_grow([6 * 10**6] * 7 + [8_050_000, 15_120_000], 2, 1)),
    "biglstm": dict(B=128, D=40_000_000, vals=_grow([10**6] * 5 + [3_200_000], 32, 10)),
}


def sweep_scenario(model, t1_ps, grad_bytes, ar_mode=0, ar_on=True):
    c = SWEEP_CURVES[model]
    G, E = _knots(c["B"], c["vals"])
    return dict(dataset_items=c["D"], mini_batch=c["B"], knot_G=G, knot_uepochs=E,
                grad_bytes=grad_bytes, t1_ps=t1_ps,
                bw_intra_Bps=900_000_000_000 if ar_on else 0, lat_intra_ps=2_000_000,
                bw_inter_Bps=50_000_000_000 if ar_on else 0, lat_inter_ps=5_000_000,
                node_size=8, ar_mode=ar_mode)


# ---- paper-anchored fixtures (AR off, SE ≡ 1 as PAPER.md:290) ------------
def inception_fixture():
    """K10: T_1 = 132u, T_2 = 100u (Table 1 1.32×), B = 64,
    D = 2^22; E = 4 up to G = 2048, 7 at 4096, 12 at 8192, 23 at 16384."""
    G = [64 * 2**k for k in range(9)]
    E = [4 * 10**6] * 6 + [7 * 10**6, 12 * 10**6, 23 * 10**6]
    sc = dict(dataset_items=2**22, mini_batch=64, knot_G=G, knot_uepochs=E, grad_bytes=0,
              t1_ps=132 * U, node_size=8, ar_mode=0)
    return sc, [1, 2], [132 * U, 100 * U], 256


def biglstm_fixture():
    """K11: T_1 = 122u, T_2 = 100u (1.22×), B = 128, D = 2^22,
    E flat to G = 2048, ×3.2 at 4096."""
    G = [128 * 2**k for k in range(6)]
    E = [10**6] * 5 + [3_200_000]
    sc = dict(dataset_items=2**22, mini_batch=128, knot_G=G, knot_uepochs=E, grad_bytes=0,
              t1_ps=122 * U, node_size=8, ar_mode=0)
    return sc, [1, 2], [122 * U, 100 * U], 32


def gnmt_fixture():
    """K12: T_1 = 115u, T_2 = 100u (1.15×), B = 128, D = 2^22,
    E_256/E_128 = 216/115 (inverting +8% @256)."""
    G = [128 * 2**k for k in range(9)]
    E = [6 * 10**6] * 7 + [8_050_000, 15_120_000]
    sc = dict(dataset_items=2**22, mini_batch=128, knot_G=G, knot_uepochs=E, grad_bytes=0,
              t1_ps=115 * U, node_size=8, ar_mode=0)
    return sc, [1, 2], [115 * U, 100 * U], 256
