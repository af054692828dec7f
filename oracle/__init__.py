"""ctypes wrapper of the CPU oracle (oracle/pp_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  It shares
no code with ``paper_1907_13257_b200`` and imports nothing from it.

Every function follows SURVEY.md §8(c) O1–O12 (the readings of PAPER.md listed
there and in DESIGN.md); see the C source for per-function citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

GEN_GRAY, GEN_RANDOM, GEN_PERTURB = 0, 1, 2
INFEASIBLE = (1 << 64) - 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, single thread)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-Wall",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class _Input(C.Structure):
    _fields_ = [("K", C.c_int32), ("E", C.c_int32),
                ("op_id", C.POINTER(C.c_int64)),
                ("fwd_ps", C.POINTER(C.c_uint64)), ("bwd_ps", C.POINTER(C.c_uint64)),
                ("mem_bytes", C.POINTER(C.c_uint64)), ("param_bytes", C.POINTER(C.c_uint64)),
                ("edge_src", C.POINTER(C.c_int32)), ("edge_dst", C.POINTER(C.c_int32)),
                ("edge_fwd_bytes", C.POINTER(C.c_uint64)), ("edge_bwd_bytes", C.POINTER(C.c_uint64)),
                ("link_bw_Bps", C.c_uint64), ("link_lat_ps", C.c_uint64),
                ("dev_mem_cap_bytes", C.c_uint64)]


class _Hw(C.Structure):
    _fields_ = [("num_devices", C.c_int32), ("num_routers", C.c_int32), ("num_links", C.c_int32),
                ("link_a", C.POINTER(C.c_int32)), ("link_b", C.POINTER(C.c_int32)),
                ("link_bw_Bps", C.POINTER(C.c_uint64)), ("link_lat_ps", C.POINTER(C.c_uint64)),
                ("dev_mem_cap_bytes", C.c_uint64)]


class _Result(C.Structure):
    _fields_ = [("best_makespan_ps", C.c_uint64), ("best_index", C.c_uint64),
                ("best_round", C.c_uint64), ("t1_ps", C.c_uint64), ("evaluated", C.c_uint64)]


class _Best(C.Structure):
    _fields_ = [("makespan", C.c_uint64), ("index", C.c_uint64)]


class _Scenario(C.Structure):
    _fields_ = [("dataset_items", C.c_uint64), ("mini_batch", C.c_uint32), ("n_knots", C.c_uint32),
                ("knot_G", C.POINTER(C.c_uint64)), ("knot_uepochs", C.POINTER(C.c_uint64)),
                ("grad_bytes", C.c_uint64),
                ("bw_intra_Bps", C.c_uint64), ("lat_intra_ps", C.c_uint64),
                ("bw_inter_Bps", C.c_uint64), ("lat_inter_ps", C.c_uint64),
                ("node_size", C.c_uint32), ("ar_mode", C.c_uint32), ("t1_ps", C.c_uint64),
                ("n_accum", C.c_uint32), ("_pad", C.c_uint32), ("accum", C.POINTER(C.c_uint32)),
                ("shard_bytes", C.POINTER(C.c_uint64))]


class Cell(C.Structure):
    _fields_ = [("C_lo", C.c_uint64), ("C_hi", C.c_uint64), ("step_ps", C.c_uint64),
                ("steps", C.c_uint64), ("uepochs", C.c_uint64), ("feasible", C.c_uint32),
                ("accum", C.c_uint32)]

    @property
    def C(self) -> int:
        return (int(self.C_hi) << 64) | int(self.C_lo)


class _Cross(C.Structure):
    _fields_ = [("n_star", C.c_uint32), ("m_at_n_star", C.c_uint32),
                ("n_star_M", C.c_uint32 * 8), ("persistent_M", C.c_uint32 * 8),
                ("n_star_vs_best_dp", C.c_uint32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        L.or_prepare.argtypes = [P(_Input), P(C.c_void_p), C.c_char_p, C.c_int]
        L.or_prepare.restype = C.c_int
        L.or_prepare_hw.argtypes = [P(_Input), P(_Hw), P(C.c_void_p), C.c_char_p, C.c_int]
        L.or_prepare_hw.restype = C.c_int
        L.or_hw_edge_cost.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
        L.or_hw_edge_cost.restype = C.c_uint64
        L.or_free.argtypes = [C.c_void_p]
        L.or_num_ops.argtypes = [C.c_void_p]
        L.or_get_pi.argtypes = [C.c_void_p, P(C.c_int32)]
        L.or_t1.argtypes = [C.c_void_p]; L.or_t1.restype = C.c_uint64
        L.or_grad_bytes.argtypes = [C.c_void_p]; L.or_grad_bytes.restype = C.c_uint64
        L.or_edge_cost.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, P(C.c_int)]
        L.or_edge_cost.restype = C.c_uint64
        L.or_schedule.argtypes = [C.c_void_p, C.c_int, P(C.c_uint8)]
        L.or_schedule.restype = C.c_uint64
        L.or_schedule_ex.argtypes = [C.c_void_p, C.c_int, P(C.c_uint8), P(C.c_uint64), P(C.c_uint64)]
        L.or_schedule_ex.restype = C.c_uint64
        L.or_makespan_orig.argtypes = [C.c_void_p, C.c_int, P(C.c_uint8), P(C.c_uint64)]
        L.or_exact.argtypes = [C.c_void_p, C.c_int, P(C.c_uint8)]
        L.or_exact.restype = C.c_uint64
        L.or_makespan_exact_orig.argtypes = [C.c_void_p, C.c_int, P(C.c_uint8), P(C.c_uint64)]
        L.or_round_exact.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint32, P(C.c_uint8),
                                     C.c_uint64, C.c_uint64]
        L.or_round_exact.restype = _Best
        L.or_eft_orig.argtypes = [C.c_void_p, C.c_int, P(C.c_uint8)]
        L.or_pipeline_ex.argtypes = [C.c_void_p, C.c_int, P(C.c_int32), C.c_uint32, C.c_uint64]
        L.or_pipeline_ex.restype = C.c_uint64
        L.or_pipeline_search_ex.argtypes = [C.c_void_p, C.c_int, P(C.c_uint32), C.c_int, C.c_uint64, C.c_uint64,
                                            C.c_uint64]
        L.or_pipeline_search_ex.restype = _Best
        L.or_shard_bytes.argtypes = [C.c_void_p, C.c_int, P(C.c_uint8), P(C.c_uint64)]
        L.or_mix.argtypes = [C.c_uint64]; L.or_mix.restype = C.c_uint64
        L.or_gen.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint32, P(C.c_uint8),
                             C.c_uint64, P(C.c_uint8)]
        L.or_gen.restype = None
        L.or_round.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint32, P(C.c_uint8),
                               C.c_uint64, C.c_uint64]
        L.or_round.restype = _Best
        L.or_search.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint32,
                                C.c_uint32, P(C.c_uint8), P(_Result), P(C.c_uint8)]
        L.or_ar64.argtypes = [P(_Scenario), C.c_uint64, C.c_uint64, P(C.c_int)]
        L.or_ar64.restype = C.c_uint64
        L.or_epochs.argtypes = [P(_Scenario), C.c_uint64, P(C.c_uint64)]
        L.or_project.argtypes = [P(_Scenario), C.c_int, P(C.c_uint32), P(C.c_uint64), C.c_uint32, P(Cell)]
        L.or_crossover.argtypes = [P(Cell), C.c_int, P(C.c_uint32), C.c_uint32, P(_Cross), P(C.c_uint32)]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


@dataclass
class SearchResult:
    best_makespan_ps: int
    best_index: int
    best_round: int
    t1_ps: int
    evaluated: int
    placement: np.ndarray  # descriptor order


class Dfg:
    """Prepared DFG (π, adjacency, edge costs).  Arrays in descriptor order."""

    def __init__(self, fwd_ps, bwd_ps, edge_src, edge_dst, edge_fwd_bytes, link_bw_Bps=1,
                 link_lat_ps=0, edge_bwd_bytes=None, op_id=None, mem_bytes=None,
                 param_bytes=None, dev_mem_cap_bytes=0, hw=None):
        self._keep = []
        fwd = _u64(fwd_ps); bwd = _u64(bwd_ps)
        K = len(fwd)
        src = np.ascontiguousarray(np.asarray(edge_src, dtype=np.int32))
        dst = np.ascontiguousarray(np.asarray(edge_dst, dtype=np.int32))
        bf = _u64(edge_fwd_bytes)
        bb = _u64(edge_bwd_bytes) if edge_bwd_bytes is not None else None
        ids = np.ascontiguousarray(np.asarray(op_id, dtype=np.int64)) if op_id is not None else None
        mem = _u64(mem_bytes) if mem_bytes is not None else None
        par = _u64(param_bytes) if param_bytes is not None else None
        self._keep = [fwd, bwd, src, dst, bf, bb, ids, mem, par]
        inp = _Input(K, len(src), _ptr(ids, C.c_int64), _ptr(fwd, C.c_uint64), _ptr(bwd, C.c_uint64),
                     _ptr(mem, C.c_uint64), _ptr(par, C.c_uint64), _ptr(src, C.c_int32),
                     _ptr(dst, C.c_int32), _ptr(bf, C.c_uint64), _ptr(bb, C.c_uint64),
                     int(link_bw_Bps), int(link_lat_ps), int(dev_mem_cap_bytes))
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        if hw is None:
            rc = lib().or_prepare(C.byref(inp), C.byref(h), err, 512)
        else:
            la = np.ascontiguousarray(np.asarray(hw["link_a"], dtype=np.int32))
            lb = np.ascontiguousarray(np.asarray(hw["link_b"], dtype=np.int32))
            bw = _u64(hw["link_bw_Bps"]); lat = _u64(hw["link_lat_ps"])
            self._keep += [la, lb, bw, lat]
            h_ = _Hw(int(hw["num_devices"]), int(hw.get("num_routers", 0)), len(la), _ptr(la, C.c_int32),
                     _ptr(lb, C.c_int32), _ptr(bw, C.c_uint64), _ptr(lat, C.c_uint64),
                     int(hw.get("dev_mem_cap_bytes", 0)))
            rc = lib().or_prepare_hw(C.byref(inp), C.byref(h_), C.byref(h), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        self._h = h
        self.K = K
        self.E = len(src)

    @classmethod
    def from_spec(cls, spec: dict) -> "Dfg":
        keys = ["fwd_ps", "bwd_ps", "edge_src", "edge_dst", "edge_fwd_bytes", "link_bw_Bps",
                "link_lat_ps", "edge_bwd_bytes", "op_id", "mem_bytes", "param_bytes",
                "dev_mem_cap_bytes", "hw"]
        return cls(**{k: spec[k] for k in keys if k in spec and spec[k] is not None})

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_free(self._h)
            self._h = None

    @property
    def pi(self) -> np.ndarray:
        out = np.zeros(self.K, dtype=np.int32)
        lib().or_get_pi(self._h, out.ctypes.data_as(C.POINTER(C.c_int32)))
        return out

    def hw_edge_cost(self, e, a, b, bwd=False) -> int:
        """c(e, a, b) of the hardware graph (0 when a == b)."""
        return int(lib().or_hw_edge_cost(self._h, e, a, b, 1 if bwd else 0))

    @property
    def t1(self) -> int:
        return int(lib().or_t1(self._h))

    @property
    def grad_bytes(self) -> int:
        return int(lib().or_grad_bytes(self._h))

    def makespan(self, M: int, placement) -> int:
        """O4 on a placement in descriptor order."""
        d = np.ascontiguousarray(np.asarray(placement, dtype=np.uint8))
        out = C.c_uint64()
        rc = lib().or_makespan_orig(self._h, M, d.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(out))
        if rc:
            raise OracleError(rc)
        return int(out.value)

    def makespan_exact(self, M: int, placement) -> int:
        """NEXT f1: the makespan-optimal schedule of a placement in descriptor order."""
        d = np.ascontiguousarray(np.asarray(placement, dtype=np.uint8))
        out = C.c_uint64()
        rc = lib().or_makespan_exact_orig(self._h, M, d.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(out))
        if rc:
            raise OracleError(rc)
        return int(out.value)

    def shard_bytes(self, M: int, placement) -> list:
        """NEXT f4: per-device gradient shard of a placement (descriptor order)."""
        d = np.ascontiguousarray(np.asarray(placement, dtype=np.uint8))
        out = np.zeros(8, dtype=np.uint64)
        rc = lib().or_shard_bytes(self._h, M, d.ctypes.data_as(C.POINTER(C.c_uint8)),
                                  out.ctypes.data_as(C.POINTER(C.c_uint64)))
        if rc:
            raise OracleError(rc)
        return [int(x) for x in out]

    def pipeline(self, M: int, cuts, micro: int, overhead=0) -> int:
        """NEXT f3: GPipe makespan of stages cut at π positions `cuts` (M−1
        increasing values in 1..K−1) with `micro` micro-batches and a per-op
        per-micro-batch overhead (ps)."""
        cu = np.ascontiguousarray(np.asarray(list(cuts) + [0], dtype=np.int32))
        return int(lib().or_pipeline_ex(self._h, M, cu.ctypes.data_as(C.POINTER(C.c_int32)), micro, overhead))

    def pipeline_search(self, M: int, micro, begin=0, end=None, overhead=0):
        """(makespan, index) over candidates [begin, end), index = rank·len(micro) + j."""
        mi = np.ascontiguousarray(np.asarray(micro, dtype=np.uint32))
        end = (1 << 64) - 1 if end is None else end
        r = lib().or_pipeline_search_ex(self._h, M, mi.ctypes.data_as(C.POINTER(C.c_uint32)), len(mi), begin, end,
                                        overhead)
        return int(r.makespan), int(r.index)

    def eft(self, M: int) -> np.ndarray:
        """NEXT f4: the EFT-greedy placement (descriptor order)."""
        d = np.zeros(self.K, dtype=np.uint8)
        rc = lib().or_eft_orig(self._h, M, d.ctypes.data_as(C.POINTER(C.c_uint8)))
        if rc:
            raise OracleError(rc)
        return d

    def exact_pi(self, M: int, d_pi) -> int:
        d = np.ascontiguousarray(np.asarray(d_pi, dtype=np.uint8))
        return int(lib().or_exact(self._h, M, d.ctypes.data_as(C.POINTER(C.c_uint8))))

    def round_exact(self, M, gen, seed_r, tau, base_pi, begin, end):
        base = np.ascontiguousarray(np.asarray(base_pi if base_pi is not None else np.zeros(self.K),
                                               dtype=np.uint8))
        r = lib().or_round_exact(self._h, M, gen, seed_r, tau, base.ctypes.data_as(C.POINTER(C.c_uint8)),
                                 begin, end)
        return int(r.makespan), int(r.index)

    def makespan_pi(self, M: int, d_pi) -> int:
        d = np.ascontiguousarray(np.asarray(d_pi, dtype=np.uint8))
        return int(lib().or_schedule(self._h, M, d.ctypes.data_as(C.POINTER(C.c_uint8))))

    def schedule(self, M: int, placement):
        """(makespan, fwd starts, bwd starts), all in descriptor order."""
        d = np.asarray(placement, dtype=np.uint8)[self.pi]
        d = np.ascontiguousarray(d)
        sf = np.zeros(self.K, dtype=np.uint64); sb = np.zeros(self.K, dtype=np.uint64)
        mk = lib().or_schedule_ex(self._h, M, d.ctypes.data_as(C.POINTER(C.c_uint8)),
                                  sf.ctypes.data_as(C.POINTER(C.c_uint64)),
                                  sb.ctypes.data_as(C.POINTER(C.c_uint64)))
        f = np.zeros(self.K, dtype=np.uint64); b = np.zeros(self.K, dtype=np.uint64)
        f[self.pi] = sf; b[self.pi] = sb
        return int(mk), f, b

    def round(self, M, gen, seed_r, tau, base_pi, begin, end):
        base = np.ascontiguousarray(np.asarray(base_pi if base_pi is not None else np.zeros(self.K),
                                               dtype=np.uint8))
        r = lib().or_round(self._h, M, gen, seed_r, tau, base.ctypes.data_as(C.POINTER(C.c_uint8)),
                           begin, end)
        return int(r.makespan), int(r.index)

    def search(self, M, gen, seed, count, rounds=1, tau=0, base=None) -> SearchResult:
        res = _Result()
        pl = np.zeros(self.K, dtype=np.uint8)
        b = None
        if base is not None:
            b = np.ascontiguousarray(np.asarray(base, dtype=np.uint8))
        rc = lib().or_search(self._h, M, gen, seed, count, rounds, tau,
                             b.ctypes.data_as(C.POINTER(C.c_uint8)) if b is not None else None,
                             C.byref(res), pl.ctypes.data_as(C.POINTER(C.c_uint8)))
        if rc:
            raise OracleError(rc)
        return SearchResult(int(res.best_makespan_ps), int(res.best_index), int(res.best_round),
                            int(res.t1_ps), int(res.evaluated), pl)


def gen(K, M, gen_kind, seed_r, tau, base_pi, i) -> np.ndarray:
    """O5/O6: candidate i's placement in π order."""
    base = np.ascontiguousarray(np.asarray(base_pi if base_pi is not None else np.zeros(K), dtype=np.uint8))
    d = np.zeros(K, dtype=np.uint8)
    lib().or_gen(K, M, gen_kind, seed_r, tau, base.ctypes.data_as(C.POINTER(C.c_uint8)), i,
                 d.ctypes.data_as(C.POINTER(C.c_uint8)))
    return d


def mix(z: int) -> int:
    return int(lib().or_mix(z))


def edge_cost(nbytes, bw, lat) -> int:
    ov = C.c_int(0)
    v = int(lib().or_edge_cost(nbytes, bw, lat, C.byref(ov)))
    if ov.value:
        raise OracleError(-3, "edge cost overflow")
    return v


class Scenario:
    """O8–O10 inputs; keeps its arrays alive."""

    def __init__(self, dataset_items, mini_batch, knot_G, knot_uepochs, grad_bytes, t1_ps,
                 bw_intra_Bps=0, lat_intra_ps=0, bw_inter_Bps=0, lat_inter_ps=0, node_size=8,
                 ar_mode=0, accum=None, shard_bytes=None):
        """accum: accumulation factors offered per cell (NEXT f4); shard_bytes:
        [nM][8] per-device gradient shards of each M's placement, or None."""
        self.kG = _u64(knot_G); self.kE = _u64(knot_uepochs)
        self.acc = np.ascontiguousarray(np.asarray(accum, dtype=np.uint32)) if accum is not None else None
        self.sh = _u64(np.asarray(shard_bytes, dtype=np.uint64).reshape(-1)) if shard_bytes is not None else None
        self.s = _Scenario(int(dataset_items), int(mini_batch), len(self.kG),
                           _ptr(self.kG, C.c_uint64), _ptr(self.kE, C.c_uint64), int(grad_bytes),
                           int(bw_intra_Bps), int(lat_intra_ps), int(bw_inter_Bps), int(lat_inter_ps),
                           int(node_size), int(ar_mode), int(t1_ps),
                           len(self.acc) if self.acc is not None else 0, 0,
                           _ptr(self.acc, C.c_uint32), _ptr(self.sh, C.c_uint64))

    @classmethod
    def from_spec(cls, spec: dict) -> "Scenario":
        return cls(**spec)

    def ar(self, n, n_devices) -> int:
        rc = C.c_int(0)
        v = int(lib().or_ar64(C.byref(self.s), n, n_devices, C.byref(rc)))
        if rc.value:
            raise OracleError(rc.value)
        return v

    def epochs(self, G):
        E = C.c_uint64()
        ok = lib().or_epochs(C.byref(self.s), G, C.byref(E))
        return int(E.value) if ok else None

    def project(self, Ms, T_M, N_max):
        nM = len(Ms)
        ms = np.ascontiguousarray(np.asarray(Ms, dtype=np.uint32))
        tm = _u64(T_M)
        cells = (Cell * (nM * N_max))()
        rc = lib().or_project(C.byref(self.s), nM, _ptr(ms, C.c_uint32), _ptr(tm, C.c_uint64),
                              N_max, cells)
        if rc:
            raise OracleError(rc)
        return cells


@dataclass
class Crossover:
    n_star: int
    m_at_n_star: int
    n_star_M: list
    persistent_M: list
    n_star_vs_best_dp: int
    best_m: list


def crossover(cells, Ms, N_max) -> Crossover:
    nM = len(Ms)
    ms = np.ascontiguousarray(np.asarray(Ms, dtype=np.uint32))
    r = _Cross()
    bm = np.zeros(N_max, dtype=np.uint32)
    rc = lib().or_crossover(cells, nM, _ptr(ms, C.c_uint32), N_max, C.byref(r),
                            bm.ctypes.data_as(C.POINTER(C.c_uint32)))
    if rc:
        raise OracleError(rc)
    return Crossover(int(r.n_star), int(r.m_at_n_star), [int(x) for x in r.n_star_M[:nM]],
                     [int(x) for x in r.persistent_M[:nM]], int(r.n_star_vs_best_dp),
                     [int(x) for x in bm])


def cell_C(cells, m, N, N_max) -> int:
    return cells[m * N_max + (N - 1)].C
