"""B200-native dynamic random-walk engine (FlexiWalker, arXiv 2512.00705).

Python binding of the C ABI in include/dynwalk_b200.h (libdynwalk_b200.so).
The compute path is the CUDA library; this module only marshals arguments.
It mirrors the reference's host API for the walk path:

    reference (/root/reference/proj)              here
    ------------------------------------------    -----------------------------
    Graph (graph.hpp:55-126) / Graph::build       DeviceGraph.from_csr / .rmat
    profile_edge_cost_ratio (cost_model.hpp:39)   profile_edge_cost_ratio
    run_queries (runtime.hpp:85-86)               run_queries
    RunOptions / RunStats / RunResult             RunOptions / dict / RunResult
    Node2Vec / MetaPath / SecondOrderPr / Static  Model(kind=...)

There is no CPU fallback: importing works anywhere, but every call that
computes goes through the CUDA library and raises if it is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = ["DeviceGraph", "Model", "RunOptions", "ProfileConfig", "RunResult", "DynwalkError", "run_queries",
           "profile_edge_cost_ratio", "tune_edge_cost_ratio", "shard_of", "library_path", "load_library", "EXPORTED_SYMBOLS",
           "INVALID_VERTEX"]

HERE = os.path.dirname(os.path.abspath(__file__))
# DYNWALK_B200_LIB selects a locally built variant (performance experiments)
LIB = os.environ.get("DYNWALK_B200_LIB", os.path.join(HERE, "lib", "libdynwalk_b200.so"))
INVALID_VERTEX = 0xFFFFFFFF

EXPORTED_SYMBOLS = (
    "dw_abi_version", "dw_last_error", "dw_device_count", "dw_graph_create", "dw_graph_load_dwg1",
    "dw_graph_generate_rmat", "dw_graph_destroy", "dw_graph_info", "dw_graph_download",
    "dw_calibrate", "dw_calibrate_ex", "dw_tune_ratio", "dw_model_compile", "dw_model_free", "dw_run", "dw_run_compact",
    "dw_run_write_paths", "dw_run_device",
    "dw_run_device_sync",
    "dw_host_alloc",
    "dw_host_free",
    "dw_selftest_math",
)

MODEL_KINDS = {"static": 0, "node2vec": 1, "metapath": 2, "pr2": 3, "custom": 4}
MODES = {"adaptive": 0, "force-ervs": 1, "force-erjs": 2, "ervs-nojump": 3, "force-its": 4,
         "force-als": 5}


class DynwalkError(RuntimeError):
    """dynwalk::Error analogue (types.hpp:17-20)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
u16p = C.POINTER(C.c_uint16)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)


class GraphDesc(C.Structure):
    _fields_ = [("num_vertices", C.c_uint32), ("num_edges", C.c_uint64),
                ("row_offsets", u64p), ("col_indices", u32p), ("edge_props", f32p),
                ("edge_labels", u16p), ("node_prop_max", f64p), ("node_prop_sum", f64p)]


class RmatDesc(C.Structure):
    _fields_ = [("scale", C.c_uint32), ("edge_factor", C.c_uint32), ("seed", C.c_uint64),
                ("weights", C.c_int), ("low", C.c_double), ("high", C.c_double),
                ("alpha", C.c_double), ("weight_seed", C.c_uint64), ("labels", C.c_int),
                ("label_low", C.c_uint32), ("label_high", C.c_uint32),
                ("label_seed", C.c_uint64)]


class ModelDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("weighted", C.c_int), ("a", C.c_double), ("b", C.c_double),
                ("gamma", C.c_double), ("schema", u16p), ("schema_len", C.c_uint32),
                ("custom", C.c_void_p)]


class RunOptsC(C.Structure):
    _fields_ = [("mode", C.c_int), ("walk_length", C.c_uint32), ("seed", C.c_uint64),
                ("erjs_cap_per_degree", C.c_uint64), ("edge_cost_ratio", C.c_double),
                ("qid_base", C.c_uint64), ("qids", C.c_void_p), ("erjs_handoff", C.c_double)]


class ProfileConfigC(C.Structure):
    _fields_ = [("node_fraction", C.c_double), ("min_nodes", C.c_uint32),
                ("neighbors_per_node", C.c_uint32), ("repetitions", C.c_uint32),
                ("seed", C.c_uint64)]


class RunStatsC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "queries", "query_errors", "dead_ends", "steps", "select_ervs", "select_erjs",
        "select_its", "select_als", "trials", "weight_reads", "rng_draws", "erjs_fallbacks")] + [
        ("selection_by_degree", (C.c_uint64 * 2) * 33), ("kernel_ms", C.c_double),
        ("total_ms", C.c_double), ("kernel_launches", C.c_uint64),
        ("algorithmic_bytes", C.c_uint64)]

    def as_dict(self) -> dict:
        d = {n: getattr(self, n) for n, _ in self._fields_ if n != "selection_by_degree"}
        d = {k: (float(v) if isinstance(v, float) else int(v)) for k, v in d.items()}
        d["selection_by_degree"] = [(int(self.selection_by_degree[b][0]),
                                     int(self.selection_by_degree[b][1])) for b in range(33)]
        return d


_lib = None


def library_path() -> str:
    return LIB


def load_library() -> C.CDLL:
    """Load libdynwalk_b200.so; raises if it was never built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        raise DynwalkError(-4, f"CUDA library missing: {LIB} (run __graft_entry__.build())")
    L = C.CDLL(LIB)
    vp = C.c_void_p
    L.dw_last_error.restype = C.c_char_p
    L.dw_abi_version.restype = C.c_int
    L.dw_device_count.argtypes = [C.POINTER(C.c_int)]
    L.dw_graph_create.argtypes = [C.POINTER(GraphDesc), C.POINTER(C.c_int), C.c_int,
                                  C.POINTER(vp)]
    L.dw_graph_generate_rmat.argtypes = [C.POINTER(RmatDesc), C.POINTER(C.c_int), C.c_int,
                                         C.POINTER(vp)]
    L.dw_graph_load_dwg1.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]
    L.dw_graph_destroy.argtypes = [vp]
    L.dw_graph_info.argtypes = [vp, u32p, u64p, C.POINTER(C.c_int), u32p]
    L.dw_graph_download.argtypes = [vp, u64p, u32p, f32p, u16p, f64p, f64p]
    L.dw_calibrate.argtypes = [vp, C.POINTER(ModelDesc), C.c_uint64, f64p]
    L.dw_calibrate_ex.argtypes = [vp, C.POINTER(ModelDesc), C.POINTER(ProfileConfigC), f64p]
    L.dw_tune_ratio.argtypes = [vp, C.POINTER(ModelDesc), C.POINTER(ProfileConfigC), C.c_uint32,
                                f64p]
    L.dw_model_compile.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.POINTER(vp)]
    L.dw_model_free.argtypes = [vp]
    L.dw_run.argtypes = [vp, C.POINTER(ModelDesc), u32p, C.c_uint64, C.POINTER(RunOptsC), u32p,
                         u32p, C.POINTER(RunStatsC)]
    L.dw_run_compact.argtypes = [vp, C.POINTER(ModelDesc), u32p, C.c_uint64,
                                 C.POINTER(RunOptsC), u64p, u32p, C.c_uint64,
                                 C.POINTER(RunStatsC)]
    L.dw_run_write_paths.argtypes = [vp, C.POINTER(ModelDesc), u32p, C.c_uint64,
                                     C.POINTER(RunOptsC), C.c_char_p, C.POINTER(RunStatsC)]
    L.dw_run_device.argtypes = [vp, C.c_int, C.POINTER(ModelDesc), vp, C.c_uint64,
                                C.POINTER(RunOptsC), vp, vp, vp]
    L.dw_run_device_sync.argtypes = [vp, C.c_int, C.POINTER(RunStatsC)]
    L.dw_host_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
    L.dw_host_free.argtypes = [vp]
    L.dw_selftest_math.argtypes = [C.c_int, f64p, f64p, C.c_uint64]
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc != 0:
        raise DynwalkError(rc, load_library().dw_last_error().decode())


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


@dataclass
class Model:
    """A builtin walk model (models.hpp:33-164)."""
    kind: str = "node2vec"
    weighted: bool = True
    a: float = 2.0
    b: float = 0.5
    gamma: float = 0.2
    schema: tuple = (0, 1, 2, 3, 4)
    custom: "CustomModel" = None  # kind "custom": a compiled DslWalk
    _arr: np.ndarray = field(default=None, repr=False)

    def c(self) -> ModelDesc:
        if self.kind not in MODEL_KINDS:
            raise DynwalkError(-1, f"unknown model '{self.kind}' (expected static, node2vec, "
                                   "metapath, pr2, custom)")
        self._arr = np.ascontiguousarray(self.schema, np.uint16)
        return ModelDesc(MODEL_KINDS[self.kind], int(self.weighted), self.a, self.b, self.gamma,
                         _p(self._arr, u16p), len(self.schema),
                         self.custom.h if self.custom is not None else None)


class CustomModel:
    """A DslWalk weight function compiled into the walk kernel (dw_model_compile).

    `source` is the CUDA model functor generated from the reference's parsed
    program by paper_2512_00705_b200/host/dsl_codegen.hpp."""

    def __init__(self, source: str, max_steps: int = 2**32 - 1, flags: int = 0):
        L = load_library()
        self.h = C.c_void_p()
        _check(L.dw_model_compile(source.encode(), max_steps, flags, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            load_library().dw_model_free(self.h)
            self.h = None


@dataclass
class RunOptions:
    """RunOptions (runtime.hpp:17-32) + CostModelParams.edge_cost_ratio."""
    mode: str = "adaptive"
    walk_length: int = 80
    seed: int = 0
    erjs_cap_per_degree: int = 64
    edge_cost_ratio: float = 1.0
    qid_base: int = 0
    # global walker ids (RNG keys) of the queries: a host uint64 array for
    # run_queries*, or an int device address for dw_run_device; None = qid_base + i
    qids: object = None
    # tier-2 eRJS hand-off (0 = the reference's rule; include/dynwalk_b200.h)
    erjs_handoff: float = 0.0

    def c(self) -> RunOptsC:
        if self.mode not in MODES:
            raise DynwalkError(-1, f"unknown sampler mode '{self.mode}'")
        q = self.qids
        if isinstance(q, np.ndarray):
            if q.dtype != np.uint64 or not q.flags.c_contiguous:
                raise DynwalkError(-1, "qids must be a contiguous uint64 array")
            q = q.ctypes.data
        return RunOptsC(MODES[self.mode], self.walk_length, self.seed & (2**64 - 1),
                        self.erjs_cap_per_degree, self.edge_cost_ratio, self.qid_base, q,
                        self.erjs_handoff)


@dataclass
class RunResult:
    paths: np.ndarray | None   # [nq][walk_length+1] uint32, INVALID padded
    lengths: np.ndarray        # [nq]; 0 = per-query error (empty path)
    stats: dict

    def path_list(self) -> list:
        """RunResult.paths as the reference returns it (vector<vector<u32>>)."""
        return [list(map(int, self.paths[i, :n])) for i, n in enumerate(self.lengths)]


class DeviceGraph:
    """Device-resident CSR replicated on `devices` (dw_graph_t)."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            load_library().dw_graph_destroy(h)
            self.h = None

    @staticmethod
    def _devs(devices):
        if devices is None:
            return None, 1
        arr = (C.c_int * len(devices))(*devices)
        return arr, len(devices)

    @classmethod
    def from_csr(cls, row, col, prop, label=None, nmax=None, nsum=None, devices=None):
        L = load_library()
        row = np.ascontiguousarray(row, np.uint64)
        col = np.ascontiguousarray(col, np.uint32)
        prop = np.ascontiguousarray(prop, np.float32)
        label = None if label is None else np.ascontiguousarray(label, np.uint16)
        nmax = None if nmax is None else np.ascontiguousarray(nmax, np.float64)
        nsum = None if nsum is None else np.ascontiguousarray(nsum, np.float64)
        d = GraphDesc(len(row) - 1, len(col), _p(row, u64p), _p(col, u32p), _p(prop, f32p),
                      _p(label, u16p), _p(nmax, f64p), _p(nsum, f64p))
        h = C.c_void_p()
        devs, nd = cls._devs(devices)
        _check(L.dw_graph_create(C.byref(d), devs, nd, C.byref(h)))
        return cls(h)

    @classmethod
    def rmat(cls, scale, edge_factor=16, seed=1, weights="uniform", low=1.0, high=5.0,
             alpha=1.0, weight_seed=2, labels=None, label_seed=3, devices=None):
        L = load_library()
        wk = {"uniform": 0, "pareto": 2, None: -1, "none": -1}[weights]
        lo, hi = labels if labels is not None else (0, 0)
        d = RmatDesc(scale, edge_factor, seed, wk, low, high, alpha, weight_seed,
                     int(labels is not None), lo, hi, label_seed)
        h = C.c_void_p()
        devs, nd = cls._devs(devices)
        _check(L.dw_graph_generate_rmat(C.byref(d), devs, nd, C.byref(h)))
        return cls(h)

    @classmethod
    def load_dwg1(cls, path: str, devices=None) -> "DeviceGraph":
        """A DWG1 binary CSR cache (dynwalk::save_binary) streamed to the devices."""
        L = load_library()
        h = C.c_void_p()
        devs, nd = cls._devs(devices)
        _check(L.dw_graph_load_dwg1(os.fsencode(path), devs, nd, C.byref(h)))
        return cls(h)

    def info(self) -> dict:
        nv, ne, hl, md = C.c_uint32(), C.c_uint64(), C.c_int(), C.c_uint32()
        _check(load_library().dw_graph_info(self.h, C.byref(nv), C.byref(ne), C.byref(hl),
                                            C.byref(md)))
        return {"num_vertices": nv.value, "num_edges": ne.value, "has_labels": bool(hl.value),
                "max_degree": md.value}

    def download(self) -> dict:
        inf = self.info()
        nv, ne = inf["num_vertices"], inf["num_edges"]
        out = {"row": np.empty(nv + 1, np.uint64), "col": np.empty(ne, np.uint32),
               "prop": np.empty(ne, np.float32), "nmax": np.empty(nv, np.float64),
               "nsum": np.empty(nv, np.float64),
               "label": np.empty(ne, np.uint16) if inf["has_labels"] else None}
        _check(load_library().dw_graph_download(
            self.h, _p(out["row"], u64p), _p(out["col"], u32p), _p(out["prop"], f32p),
            _p(out["label"], u16p), _p(out["nmax"], f64p), _p(out["nsum"], f64p)))
        return out


@dataclass
class ProfileConfig:
    """ProfileConfig (cost_model.hpp:9-15)."""
    node_fraction: float = 0.01
    min_nodes: int = 64
    neighbors_per_node: int = 32
    repetitions: int = 5
    seed: int = 0

    def c(self) -> ProfileConfigC:
        return ProfileConfigC(self.node_fraction, self.min_nodes, self.neighbors_per_node,
                              self.repetitions, self.seed)


def profile_edge_cost_ratio(g: DeviceGraph, model: Model, seed: int = 0,
                            cfg: ProfileConfig | None = None) -> float:
    """profile_edge_cost_ratio (cost_model.cpp:37-126), timed on the device.
    `cfg` overrides the ProfileConfig defaults (its seed wins over `seed`)."""
    r = C.c_double()
    m = model.c()
    c = (cfg if cfg is not None else ProfileConfig(seed=seed)).c()
    _check(load_library().dw_calibrate_ex(g.h, C.byref(m), C.byref(c), C.byref(r)))
    return r.value


def _check_qids(opts: RunOptions, nq: int) -> None:
    if isinstance(opts.qids, np.ndarray) and len(opts.qids) != nq:
        raise DynwalkError(-1, f"qids holds {len(opts.qids)} walker ids for {nq} queries")


def shard_of(qids, world: int) -> np.ndarray:
    """Rank that walks each global walker id in a `world`-way partitioned run:
    Fibonacci hashing (high 32 bits of q * 0x9E3779B97F4A7C15 mod 2^64, mod
    world).  Consecutive ids spread over all ranks, so a hub-heavy stretch of
    the query list does not land on one GPU (range partitioning scales worse,
    PAPER.md:1086).  bench.py computes the same function on the device."""
    q = np.asarray(qids, np.uint64)
    with np.errstate(over="ignore"):
        h = (q * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(32)
    return (h % np.uint64(world)).astype(np.int64)


def tune_edge_cost_ratio(g: DeviceGraph, model: Model, seed: int = 0,
                         cfg: ProfileConfig | None = None, walk_length: int = 80) -> float:
    """dw_tune_ratio: the micro-pass ratio refined by timing the walk kernel
    itself at a few thresholds around it (see include/dynwalk_b200.h)."""
    r = C.c_double()
    m = model.c()
    c = (cfg if cfg is not None else ProfileConfig(seed=seed)).c()
    _check(load_library().dw_tune_ratio(g.h, C.byref(m), C.byref(c), walk_length, C.byref(r)))
    return r.value


def run_queries(g: DeviceGraph, model: Model, queries, opts: RunOptions,
                keep_paths: bool = True, out_paths: np.ndarray | None = None) -> RunResult:
    """run_queries (runtime.cpp:192-247) on the device replicas of `g`."""
    L = load_library()
    q = np.ascontiguousarray(queries, np.uint32)
    _check_qids(opts, len(q))
    stride = opts.walk_length + 1
    paths = out_paths
    if paths is None and keep_paths:
        paths = np.empty((len(q), stride), np.uint32)
    lengths = np.empty(len(q), np.uint32)
    st = RunStatsC()
    m = model.c()
    o = opts.c()
    _check(L.dw_run(g.h, C.byref(m), _p(q, u32p), len(q), C.byref(o), _p(paths, u32p),
                    _p(lengths, u32p), C.byref(st)))
    return RunResult(paths, lengths, st.as_dict())


def run_queries_compact(g: DeviceGraph, model: Model, queries, opts: RunOptions):
    """run_queries with the RunResult.paths layout flattened (dw_run_compact):
    returns (offsets[nq+1] u64, flat u32, stats); path i is
    flat[offsets[i]:offsets[i+1]]."""
    L = load_library()
    q = np.ascontiguousarray(queries, np.uint32)
    _check_qids(opts, len(q))
    offsets = np.empty(len(q) + 1, np.uint64)
    cap = len(q) * (opts.walk_length + 1)
    flat = np.empty(max(cap, 1), np.uint32)
    st = RunStatsC()
    m = model.c()
    o = opts.c()
    _check(L.dw_run_compact(g.h, C.byref(m), _p(q, u32p), len(q), C.byref(o),
                            _p(offsets, u64p), _p(flat, u32p), cap, C.byref(st)))
    return offsets, flat[:int(offsets[-1])], st.as_dict()


def run_write_paths(g: DeviceGraph, model: Model, queries, opts: RunOptions, path: str) -> dict:
    """run_queries + write_paths (runtime.cpp:280-291) streamed to `path`, the
    text formatted on the device; returns the RunStats counters."""
    L = load_library()
    q = np.ascontiguousarray(queries, np.uint32)
    _check_qids(opts, len(q))
    st = RunStatsC()
    m = model.c()
    o = opts.c()
    _check(L.dw_run_write_paths(g.h, C.byref(m), _p(q, u32p), len(q), C.byref(o),
                                os.fsencode(path), C.byref(st)))
    return st.as_dict()
