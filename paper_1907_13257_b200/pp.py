"""Thin ctypes binding of libpp.so (include/pp.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; PyTorch only
provides device memory (tensor.data_ptr()), streams
(torch.cuda.current_stream().cuda_stream) and process groups (NCCL unique-id
exchange).  There is no CPU fallback: if libpp.so is missing or no CUDA
device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpp.so")

PP_OK = 0
ERRORS = {-1: "PP_E_INVALID", -2: "PP_E_CYCLE", -3: "PP_E_RANGE", -4: "PP_E_TOO_LARGE",
          -5: "PP_E_INFEASIBLE", -6: "PP_E_CUDA", -7: "PP_E_NCCL"}
GEN_GRAY, GEN_RANDOM, GEN_PERTURB = 0, 1, 2
TIER_SHARED, TIER_GLOBAL = 0, 1   # pp_dfg_get_tier (pp.h)
INFEASIBLE = (1 << 64) - 1


class PPError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


P = C.POINTER


class DfgDesc(C.Structure):
    _fields_ = [("num_ops", C.c_int32), ("num_edges", C.c_int32), ("op_id", P(C.c_int64)),
                ("fwd_ps", P(C.c_uint64)), ("bwd_ps", P(C.c_uint64)), ("mem_bytes", P(C.c_uint64)),
                ("param_bytes", P(C.c_uint64)), ("edge_src", P(C.c_int32)), ("edge_dst", P(C.c_int32)),
                ("edge_fwd_bytes", P(C.c_uint64)), ("edge_bwd_bytes", P(C.c_uint64))]


class LinkDesc(C.Structure):
    _fields_ = [("link_bw_Bps", C.c_uint64), ("link_lat_ps", C.c_uint64), ("dev_mem_cap_bytes", C.c_uint64)]


class HwDesc(C.Structure):
    _fields_ = [("num_devices", C.c_int32), ("num_routers", C.c_int32), ("num_links", C.c_int32),
                ("link_a", P(C.c_int32)), ("link_b", P(C.c_int32)), ("link_bw_Bps", P(C.c_uint64)),
                ("link_lat_ps", P(C.c_uint64)), ("dev_mem_cap_bytes", C.c_uint64)]


class DfgInfo(C.Structure):
    _fields_ = [("num_ops", C.c_int32), ("num_edges", C.c_int32), ("num_slots", C.c_int32),
                ("image_bytes", C.c_int32), ("t1_ps", C.c_uint64), ("grad_bytes", C.c_uint64)]


class SearchDesc(C.Structure):
    _fields_ = [("gen", C.c_int32), ("rounds", C.c_uint32), ("seed", C.c_uint64), ("count", C.c_uint64),
                ("flip_thresh", C.c_uint32), ("_pad", C.c_uint32), ("base", P(C.c_uint8))]


class SearchResultC(C.Structure):
    _fields_ = [("best_makespan_ps", C.c_uint64), ("best_index", C.c_uint64), ("best_round", C.c_uint64),
                ("t1_ps", C.c_uint64), ("evaluated", C.c_uint64), ("placement", P(C.c_uint8))]


class Scenario(C.Structure):
    _fields_ = [("dataset_items", C.c_uint64), ("mini_batch", C.c_uint32), ("n_knots", C.c_uint32),
                ("knot_G", P(C.c_uint64)), ("knot_uepochs", P(C.c_uint64)), ("grad_bytes", C.c_uint64),
                ("bw_intra_Bps", C.c_uint64), ("lat_intra_ps", C.c_uint64), ("bw_inter_Bps", C.c_uint64),
                ("lat_inter_ps", C.c_uint64), ("node_size", C.c_uint32), ("ar_mode", C.c_uint32),
                ("t1_ps", C.c_uint64), ("n_accum", C.c_uint32), ("_pad", C.c_uint32),
                ("accum", P(C.c_uint32)), ("shard_bytes", P(C.c_uint64))]


class Cell(C.Structure):
    _fields_ = [("C_lo", C.c_uint64), ("C_hi", C.c_uint64), ("step_ps", C.c_uint64), ("steps", C.c_uint64),
                ("uepochs", C.c_uint64), ("feasible", C.c_uint32), ("accum", C.c_uint32)]


CELL_BYTES = C.sizeof(Cell)   # 48


class CrossoverC(C.Structure):
    _fields_ = [("n_star", C.c_uint32), ("m_at_n_star", C.c_uint32), ("n_star_M", C.c_uint32 * 8),
                ("persistent_M", C.c_uint32 * 8), ("n_star_vs_best_dp", C.c_uint32)]


class PipelineResultC(C.Structure):
    _fields_ = [("makespan_ps", C.c_uint64), ("index", C.c_uint64), ("candidates", C.c_uint64),
                ("micro_batches", C.c_uint32), ("n_stages", C.c_uint32), ("cuts", C.c_int32 * 8)]


# exported symbol → (argtypes, restype); the C-ABI load test checks this list
# against include/pp.h
SIGNATURES = {
    "pp_load_dfg": ([P(DfgDesc), P(LinkDesc), C.c_int, P(C.c_void_p)], C.c_int),
    "pp_load_dfg_hw": ([P(DfgDesc), P(HwDesc), C.c_int, P(C.c_void_p)], C.c_int),
    "pp_free_dfg": ([C.c_void_p], None),
    "pp_dfg_get_info": ([C.c_void_p, P(DfgInfo)], C.c_int),
    "pp_dfg_get_pi": ([C.c_void_p, P(C.c_int32)], C.c_int),
    "pp_dfg_get_tier": ([C.c_void_p], C.c_int),
    "pp_plan_dfg": ([P(DfgDesc), P(LinkDesc), P(DfgInfo), P(C.c_int32)], C.c_int),
    "pp_eval_placements": ([C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p], C.c_int),
    "pp_eval_generated": ([C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint32, C.c_void_p, C.c_uint64,
                           C.c_uint64, C.c_void_p, C.c_void_p], C.c_int),
    "pp_search_range": ([C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint32, C.c_void_p, C.c_uint64,
                         C.c_uint64, C.c_void_p, C.c_void_p], C.c_int),
    "pp_eval_exact": ([C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                       C.c_void_p], C.c_int),
    "pp_eval_exact_generated": ([C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint32, C.c_void_p, C.c_uint64,
                                 C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "pp_search_exact": ([C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint32, C.c_void_p, C.c_uint64,
                         C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p], C.c_int),
    "pp_pipeline_space": ([C.c_void_p, C.c_int, C.c_int, P(C.c_uint64)], C.c_int),
    "pp_pipeline_range": ([C.c_void_p, C.c_int, P(C.c_uint32), C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                           C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "pp_pipeline_search": ([C.c_void_p, C.c_int, P(C.c_uint32), C.c_int, C.c_uint64, C.c_void_p,
                            P(PipelineResultC)], C.c_int),
    "pp_shard_bytes": ([C.c_void_p, C.c_int, P(C.c_uint8), P(C.c_uint64)], C.c_int),
    "pp_eft_place": ([C.c_void_p, C.c_int, P(C.c_uint8), C.c_void_p], C.c_int),
    "pp_search_best": ([C.c_void_p, C.c_int, P(SearchDesc), C.c_void_p, C.c_void_p, P(SearchResultC)], C.c_int),
    "pp_comm_get_unique_id": ([P(C.c_uint8)], C.c_int),
    "pp_comm_init": ([P(C.c_uint8), C.c_int, C.c_int, C.c_int, P(C.c_void_p)], C.c_int),
    "pp_comm_destroy": ([C.c_void_p], None),
    "pp_argmin_allreduce": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "pp_rank_slice": ([C.c_uint64, C.c_int, C.c_int, P(C.c_uint64), P(C.c_uint64)], None),
    "pp_comm_set_timeout": ([C.c_void_p, C.c_uint64], C.c_int),
    "pp_round_key": ([C.c_uint64, C.c_uint64, C.c_int], C.c_uint64),
    "pp_round_contrib": ([C.c_uint64, C.c_uint64, C.c_uint64], C.c_uint64),
    "pp_round_moves_base": ([C.c_uint64], C.c_int),
    "pp_round_exchange_host": ([C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, P(C.c_uint64)], C.c_int),
    "pp_pack_key": ([C.c_uint64, C.c_int], C.c_uint64),
    "pp_key_makespan": ([C.c_uint64], C.c_uint64),
    "pp_key_rank": ([C.c_uint64], C.c_int),
    "pp_project_e2e": ([P(Scenario), C.c_int, P(C.c_uint32), P(C.c_uint64), C.c_uint32, C.c_void_p,
                        C.c_void_p], C.c_int),
    "pp_crossover": ([C.c_void_p, C.c_int, P(C.c_uint32), C.c_uint32, P(CrossoverC), C.c_void_p, C.c_void_p],
                     C.c_int),
    "pp_last_error": ([], C.c_char_p),
    "pp_kernel_launch_count": ([], C.c_uint64),
    "pp_set_kernel_timing": ([C.c_int], None),
    "pp_get_kernel_timing": ([P(C.c_double), P(C.c_uint64)], None),
}

_lib = None


def lib():
    """Loads libpp.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(python -m paper_1907_13257_b200._build)")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(rc):
    if rc != PP_OK:
        raise PPError(rc, lib().pp_last_error().decode())


def _u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _ptr(a, ct):
    return a.ctypes.data_as(P(ct)) if a is not None else None


def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def _dptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _require_cuda(t, dtype_names):
    if not t.is_cuda:
        raise PPError(-1, "tensor must be on a CUDA device (no CPU fallback)")
    if str(t.dtype).split(".")[-1] not in dtype_names:
        raise PPError(-1, f"tensor dtype must be one of {dtype_names}")
    if not t.is_contiguous():
        raise PPError(-1, "tensor must be contiguous")


@dataclass
class SearchResult:
    best_makespan_ps: int
    best_index: int
    best_round: int
    t1_ps: int
    evaluated: int
    placement: np.ndarray

    @property
    def su_mp(self) -> float:
        """SU_MP(M) = T_1 / T_M, display only."""
        return self.t1_ps / self.best_makespan_ps


class Dfg:
    """A DFG resident on one GPU (pp_load_dfg).  `spec` is a dict as built by
    synth/ (descriptor-order arrays plus link parameters)."""

    def __init__(self, spec: dict, device: int = 0):
        K = len(spec["fwd_ps"])
        self._arr = dict(
            fwd=_u64(spec["fwd_ps"]), bwd=_u64(spec["bwd_ps"]),
            src=np.ascontiguousarray(np.asarray(spec["edge_src"], dtype=np.int32)),
            dst=np.ascontiguousarray(np.asarray(spec["edge_dst"], dtype=np.int32)),
            bf=_u64(spec["edge_fwd_bytes"]),
            bb=_u64(spec["edge_bwd_bytes"]) if spec.get("edge_bwd_bytes") is not None else None,
            ids=np.ascontiguousarray(np.asarray(spec["op_id"], dtype=np.int64)) if spec.get("op_id") is not None else None,
            mem=_u64(spec["mem_bytes"]) if spec.get("mem_bytes") is not None else None,
            par=_u64(spec["param_bytes"]) if spec.get("param_bytes") is not None else None)
        a = self._arr
        desc = DfgDesc(K, len(a["src"]), _ptr(a["ids"], C.c_int64), _ptr(a["fwd"], C.c_uint64),
                       _ptr(a["bwd"], C.c_uint64), _ptr(a["mem"], C.c_uint64), _ptr(a["par"], C.c_uint64),
                       _ptr(a["src"], C.c_int32), _ptr(a["dst"], C.c_int32), _ptr(a["bf"], C.c_uint64),
                       _ptr(a["bb"], C.c_uint64))
        h = C.c_void_p()
        hw = spec.get("hw")
        if hw is None:
            link = LinkDesc(int(spec["link_bw_Bps"]), int(spec["link_lat_ps"]), int(spec.get("dev_mem_cap_bytes") or 0))
            _check(lib().pp_load_dfg(C.byref(desc), C.byref(link), device, C.byref(h)))
        else:   # general hardware graph
            a.update(la=np.ascontiguousarray(np.asarray(hw["link_a"], dtype=np.int32)),
                     lb=np.ascontiguousarray(np.asarray(hw["link_b"], dtype=np.int32)),
                     hbw=_u64(hw["link_bw_Bps"]), hlat=_u64(hw["link_lat_ps"]))
            hd = HwDesc(int(hw["num_devices"]), int(hw.get("num_routers", 0)), len(a["la"]),
                        _ptr(a["la"], C.c_int32), _ptr(a["lb"], C.c_int32), _ptr(a["hbw"], C.c_uint64),
                        _ptr(a["hlat"], C.c_uint64), int(hw.get("dev_mem_cap_bytes", 0)))
            _check(lib().pp_load_dfg_hw(C.byref(desc), C.byref(hd), device, C.byref(h)))
        self._h = h
        self.device = device
        info = DfgInfo()
        _check(lib().pp_dfg_get_info(h, C.byref(info)))
        self.K, self.E, self.W = info.num_ops, info.num_edges, info.num_slots
        self.image_bytes, self.t1, self.grad_bytes = info.image_bytes, int(info.t1_ps), int(info.grad_bytes)
        self.tier = lib().pp_dfg_get_tier(h)   # TIER_SHARED / TIER_GLOBAL (pp.h)
        pi = np.zeros(K, dtype=np.int32)
        _check(lib().pp_dfg_get_pi(h, _ptr(pi, C.c_int32)))
        self.pi = pi

    def close(self):
        if getattr(self, "_h", None):
            lib().pp_free_dfg(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --------------------------------------------------------------- eval
    def eval_placements(self, M, placements, out=None, stream=None):
        """placements: uint8 CUDA tensor [count, K] (descriptor order).
        Returns an int64 CUDA tensor holding the u64 makespans bit for bit."""
        import torch
        _require_cuda(placements, ("uint8",))
        count = placements.shape[0]
        if placements.dim() != 2 or placements.shape[1] != self.K:
            raise PPError(-1, "placements must be [count, K]")
        if out is None:
            out = torch.empty(count, dtype=torch.int64, device=placements.device)
        _check(lib().pp_eval_placements(self._h, M, _dptr(placements), count, _dptr(out), _stream(stream)))
        return out

    def eval_generated(self, M, gen, seed_r, tau, base_pi, begin, count, out=None, stream=None):
        import torch
        dev = torch.device("cuda", self.device)
        if out is None:
            out = torch.empty(count, dtype=torch.int64, device=dev)
        b = None
        if gen == GEN_PERTURB:
            b = torch.as_tensor(np.asarray(base_pi, dtype=np.uint8), device=dev)
        _check(lib().pp_eval_generated(self._h, M, gen, seed_r, tau, _dptr(b), begin, count, _dptr(out),
                                       _stream(stream)))
        return out

    def search_range(self, M, gen, seed_r, tau, base_pi, begin, end, out=None, stream=None):
        """Device argmin over [begin, end): returns an int64[2] CUDA tensor
        {makespan, index} (u64 bits)."""
        import torch
        dev = torch.device("cuda", self.device)
        if out is None:
            out = torch.empty(2, dtype=torch.int64, device=dev)
        b = None
        if gen == GEN_PERTURB:
            b = torch.as_tensor(np.asarray(base_pi, dtype=np.uint8), device=dev)
        _check(lib().pp_search_range(self._h, M, gen, seed_r, tau, _dptr(b), begin, end, _dptr(out),
                                     _stream(stream)))
        return out

    # ------------------------------------------ pipeline MP (§8(f) f3)
    def pipeline_space(self, M, nm) -> int:
        c = C.c_uint64()
        _check(lib().pp_pipeline_space(self._h, M, nm, C.byref(c)))
        return int(c.value)

    def pipeline_search(self, M, micro, overhead=0, stream=None) -> dict:
        mi = np.ascontiguousarray(np.asarray(micro, dtype=np.uint32))
        r = PipelineResultC()
        _check(lib().pp_pipeline_search(self._h, M, _ptr(mi, C.c_uint32), len(mi), overhead, _stream(stream),
                                        C.byref(r)))
        return {"makespan_ps": int(r.makespan_ps), "index": int(r.index), "candidates": int(r.candidates),
                "micro_batches": int(r.micro_batches), "cuts": [int(x) for x in r.cuts[:M - 1]]}

    def pipeline_range(self, M, micro, begin, end, all_values=False, overhead=0, stream=None):
        """(makespan, index) argmin over [begin, end) — and the per-candidate
        makespans (int64 CUDA tensor) when all_values."""
        import torch
        dev = torch.device("cuda", self.device)
        mi = np.ascontiguousarray(np.asarray(micro, dtype=np.uint32))
        best = torch.empty(2, dtype=torch.int64, device=dev)
        vals = torch.empty(end - begin, dtype=torch.int64, device=dev) if all_values else None
        _check(lib().pp_pipeline_range(self._h, M, _ptr(mi, C.c_uint32), len(mi), overhead, begin, end,
                                       _dptr(best), _dptr(vals), _stream(stream)))
        b = u64(best)
        return (int(b[0]), int(b[1])), vals

    def shard_bytes(self, M, placement) -> list:
        """Per-device gradient shard S_d of a placement (descriptor order)."""
        pl = np.ascontiguousarray(np.asarray(placement, dtype=np.uint8))
        out = np.zeros(8, dtype=np.uint64)
        _check(lib().pp_shard_bytes(self._h, M, _ptr(pl, C.c_uint8), _ptr(out, C.c_uint64)))
        return [int(x) for x in out]

    def eft_place(self, M, stream=None) -> np.ndarray:
        """EFT-greedy placement (descriptor order), computed on the GPU."""
        pl = np.zeros(self.K, dtype=np.uint8)
        _check(lib().pp_eft_place(self._h, M, _ptr(pl, C.c_uint8), _stream(stream)))
        return pl

    # ------------------------------------------- exact schedule (§8(f) f1)
    def eval_exact(self, M, placements, node_limit=0, out=None, exact=None, stream=None):
        """Makespan-optimal schedule of each placement (uint8 CUDA tensor
        [count, K], descriptor order).  Returns (makespans int64 tensor,
        exact-flag uint8 tensor)."""
        import torch
        _require_cuda(placements, ("uint8",))
        count = placements.shape[0]
        if placements.dim() != 2 or placements.shape[1] != self.K:
            raise PPError(-1, "placements must be [count, K]")
        if out is None:
            out = torch.empty(count, dtype=torch.int64, device=placements.device)
        if exact is None:
            exact = torch.empty(count, dtype=torch.uint8, device=placements.device)
        _check(lib().pp_eval_exact(self._h, M, _dptr(placements), count, node_limit, _dptr(out), _dptr(exact),
                                   _stream(stream)))
        return out, exact

    def eval_exact_generated(self, M, gen, seed_r, tau, base_pi, begin, count, node_limit=0, stream=None):
        import torch
        dev = torch.device("cuda", self.device)
        out = torch.empty(count, dtype=torch.int64, device=dev)
        exact = torch.empty(count, dtype=torch.uint8, device=dev)
        b = None
        if gen == GEN_PERTURB:
            b = torch.as_tensor(np.asarray(base_pi, dtype=np.uint8), device=dev)
        _check(lib().pp_eval_exact_generated(self._h, M, gen, seed_r, tau, _dptr(b), begin, count, node_limit,
                                             _dptr(out), _dptr(exact), _stream(stream)))
        return out, exact

    def search_exact(self, M, gen, seed_r, tau, base_pi, begin, end, node_limit=0, stream=None):
        """(exact makespan, index, unresolved) of the argmin over [begin, end)."""
        import torch
        dev = torch.device("cuda", self.device)
        out = torch.empty(3, dtype=torch.int64, device=dev)
        b = None
        if gen == GEN_PERTURB:
            b = torch.as_tensor(np.asarray(base_pi, dtype=np.uint8), device=dev)
        _check(lib().pp_search_exact(self._h, M, gen, seed_r, tau, _dptr(b), begin, end, node_limit, _dptr(out),
                                     _stream(stream)))
        r = u64(out)
        return int(r[0]), int(r[1]), int(r[2])

    def search_best(self, M, gen, seed, count, rounds=1, tau=0, base=None, comm=None, stream=None):
        b = None
        if base is not None:
            b = np.ascontiguousarray(np.asarray(base, dtype=np.uint8))
        desc = SearchDesc(gen, rounds, seed, count, tau, 0, _ptr(b, C.c_uint8))
        pl = np.zeros(self.K, dtype=np.uint8)
        res = SearchResultC(0, 0, 0, 0, 0, _ptr(pl, C.c_uint8))
        _check(lib().pp_search_best(self._h, M, C.byref(desc), comm._h if comm is not None else None,
                                    _stream(stream), C.byref(res)))
        return SearchResult(int(res.best_makespan_ps), int(res.best_index), int(res.best_round),
                            int(res.t1_ps), int(res.evaluated), pl)


def plan(spec: dict) -> dict:
    """Host-only dry run of pp_load_dfg (pp_plan_dfg): K, E, the live slots W,
    the image bytes, T_1, Σ param_bytes and the state tier, with no device."""
    K = len(spec["fwd_ps"])
    fwd, bwd = _u64(spec["fwd_ps"]), _u64(spec["bwd_ps"])
    src = np.ascontiguousarray(np.asarray(spec["edge_src"], dtype=np.int32))
    dst = np.ascontiguousarray(np.asarray(spec["edge_dst"], dtype=np.int32))
    bf = _u64(spec["edge_fwd_bytes"])
    bb = _u64(spec["edge_bwd_bytes"]) if spec.get("edge_bwd_bytes") is not None else None
    ids = np.ascontiguousarray(np.asarray(spec["op_id"], dtype=np.int64)) if spec.get("op_id") is not None else None
    mem = _u64(spec["mem_bytes"]) if spec.get("mem_bytes") is not None else None
    par = _u64(spec["param_bytes"]) if spec.get("param_bytes") is not None else None
    desc = DfgDesc(K, len(src), _ptr(ids, C.c_int64), _ptr(fwd, C.c_uint64), _ptr(bwd, C.c_uint64),
                   _ptr(mem, C.c_uint64), _ptr(par, C.c_uint64), _ptr(src, C.c_int32), _ptr(dst, C.c_int32),
                   _ptr(bf, C.c_uint64), _ptr(bb, C.c_uint64))
    link = LinkDesc(int(spec["link_bw_Bps"]), int(spec["link_lat_ps"]), int(spec.get("dev_mem_cap_bytes") or 0))
    info, tier = DfgInfo(), C.c_int32()
    _check(lib().pp_plan_dfg(C.byref(desc), C.byref(link), C.byref(info), C.byref(tier)))
    return {"K": info.num_ops, "E": info.num_edges, "W": info.num_slots, "image_bytes": info.image_bytes,
            "t1": int(info.t1_ps), "grad_bytes": int(info.grad_bytes), "tier": tier.value}


# ------------------------------------------------------------ multi-GPU
class Comm:
    """NCCL communicator over the ranks of a torch.distributed process group
    (the group only carries the 128-byte unique id)."""

    def __init__(self, rank, world, device, group=None):
        uid = (C.c_uint8 * 128).from_buffer_copy(exchange_unique_id(rank, group))
        h = C.c_void_p()
        _check(lib().pp_comm_init(uid, rank, world, device, C.byref(h)))
        self._h = h
        self.rank, self.world = rank, world

    def argmin_allreduce(self, dfg, best, stream=None):
        """In place: best (int64[2] CUDA tensor {makespan, index} over this
        rank's slice) becomes the global lexicographic argmin."""
        _check(lib().pp_argmin_allreduce(dfg._h, self._h, _dptr(best), _stream(stream)))
        return best

    def set_timeout(self, ms):
        _check(lib().pp_comm_set_timeout(self._h, ms))

    def close(self):
        if getattr(self, "_h", None):
            lib().pp_comm_destroy(self._h)
            self._h = None


def exchange_unique_id(rank, group=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id; a torch.distributed
    broadcast (any backend) hands it to every rank."""
    import torch.distributed as dist
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        _check(lib().pp_comm_get_unique_id(uid))
    obj = [bytes(uid)]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def rank_slice(count, rank, world):
    b, e = C.c_uint64(), C.c_uint64()
    lib().pp_rank_slice(count, rank, world, C.byref(b), C.byref(e))
    return int(b.value), int(e.value)


def pack_key(makespan, rank):
    return int(lib().pp_pack_key(makespan, rank))


def round_key(makespan, index, rank):
    return int(lib().pp_round_key(makespan, index, rank))


def round_contrib(key_global, key_local, local_index):
    return int(lib().pp_round_contrib(key_global, key_local, local_index))


def round_moves_base(win_index) -> bool:
    return bool(lib().pp_round_moves_base(win_index))


ALLREDUCE_MIN_U64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, P(C.c_uint64))


def round_exchange_host(local_makespan, local_index, rank, allreduce_min):
    """One round's cross-rank argmin exchange run by the library's own protocol
    code (csrc/protocol.h) with a host collective: allreduce_min(int) -> int
    must return the minimum over ranks (e.g. torch.distributed over gloo).
    Returns (makespan, index) of the global winner."""
    def cb(_ctx, x, out):
        try:
            out[0] = int(allreduce_min(int(x)))
            return 0
        except Exception:   # reported as PP_E_NCCL by the library
            return 1
    fn = ALLREDUCE_MIN_U64(cb)
    win = (C.c_uint64 * 2)()
    _check(lib().pp_round_exchange_host(local_makespan, local_index, rank, C.cast(fn, C.c_void_p), None, win))
    return int(win[0]), int(win[1])


def key_makespan(key):
    return int(lib().pp_key_makespan(key))


def key_rank(key):
    return int(lib().pp_key_rank(key))


def kernel_launch_count() -> int:
    return int(lib().pp_kernel_launch_count())


def set_kernel_timing(enable: bool) -> None:
    lib().pp_set_kernel_timing(1 if enable else 0)


def get_kernel_timing():
    """(total ms, launches) of the search kernel inside search_best since enabling."""
    ms, n = C.c_double(), C.c_uint64()
    lib().pp_get_kernel_timing(C.byref(ms), C.byref(n))
    return float(ms.value), int(n.value)


# ------------------------------------------------------------ projection
def _scenario(spec):
    kG, kE = _u64(spec["knot_G"]), _u64(spec["knot_uepochs"])
    acc = spec.get("accum")
    acc = np.ascontiguousarray(np.asarray(acc, dtype=np.uint32)) if acc is not None else None
    sh = spec.get("shard_bytes")
    sh = _u64(np.asarray(sh, dtype=np.uint64).reshape(-1)) if sh is not None else None
    s = Scenario(int(spec["dataset_items"]), int(spec["mini_batch"]), len(kG), _ptr(kG, C.c_uint64),
                 _ptr(kE, C.c_uint64), int(spec.get("grad_bytes", 0)), int(spec.get("bw_intra_Bps", 0)),
                 int(spec.get("lat_intra_ps", 0)), int(spec.get("bw_inter_Bps", 0)),
                 int(spec.get("lat_inter_ps", 0)), int(spec.get("node_size", 8)), int(spec.get("ar_mode", 0)),
                 int(spec["t1_ps"]), len(acc) if acc is not None else 0, 0, _ptr(acc, C.c_uint32),
                 _ptr(sh, C.c_uint64))
    return s, (kG, kE, acc, sh)


def project_e2e(spec, Ms, T_M, N_max, cells=None, device=0, stream=None):
    """Returns a uint8 CUDA tensor [len(Ms), N_max, 48] of pp_cell records."""
    import torch
    s, keep = _scenario(spec)
    ms = np.ascontiguousarray(np.asarray(Ms, dtype=np.uint32))
    tm = _u64(T_M)
    if cells is None:
        cells = torch.empty((len(Ms), N_max, CELL_BYTES), dtype=torch.uint8, device=torch.device("cuda", device))
    _check(lib().pp_project_e2e(C.byref(s), len(Ms), _ptr(ms, C.c_uint32), _ptr(tm, C.c_uint64), N_max,
                                _dptr(cells), _stream(stream)))
    return cells


@dataclass
class Crossover:
    n_star: int
    m_at_n_star: int
    n_star_M: list
    persistent_M: list
    n_star_vs_best_dp: int
    best_m: list = field(default_factory=list)


def crossover(cells, Ms, N_max, best_m=True, stream=None):
    import torch
    ms = np.ascontiguousarray(np.asarray(Ms, dtype=np.uint32))
    r = CrossoverC()
    bm = torch.zeros(N_max, dtype=torch.int32, device=cells.device) if best_m else None
    _check(lib().pp_crossover(_dptr(cells), len(Ms), _ptr(ms, C.c_uint32), N_max, C.byref(r), _dptr(bm),
                              _stream(stream)))
    nM = len(Ms)
    return Crossover(int(r.n_star), int(r.m_at_n_star), [int(x) for x in r.n_star_M[:nM]],
                     [int(x) for x in r.persistent_M[:nM]], int(r.n_star_vs_best_dp),
                     bm.cpu().tolist() if bm is not None else [])


def cells_to_numpy(cells) -> np.ndarray:
    """pp_cell records → structured numpy array (host copy)."""
    dt = np.dtype([("C_lo", "<u8"), ("C_hi", "<u8"), ("step_ps", "<u8"), ("steps", "<u8"),
                   ("uepochs", "<u8"), ("feasible", "<u4"), ("accum", "<u4")])
    raw = cells.cpu().numpy().reshape(-1, CELL_BYTES)
    return raw.view(dt).reshape(cells.shape[0], cells.shape[1])


def u64(t) -> np.ndarray:
    """int64 CUDA tensor holding u64 bits → numpy uint64."""
    return t.cpu().numpy().view(np.uint64)
