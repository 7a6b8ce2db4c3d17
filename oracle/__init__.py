"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE ONLY).

`liboracle.so` is the C restatement of the reference walk path (oracle.c);
`_ref/libdynwalk_ref.so` is the reference's own sources compiled in place plus
ref_harness.cpp.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
import this package; the product (paper_2512_00705_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libdynwalk_ref.so")
INVALID = 0xFFFFFFFF

MODEL_KINDS = {"static": 0, "node2vec": 1, "metapath": 2, "pr2": 3, "dsl": 4}
MODES = {"adaptive": 0, "force-ervs": 1, "force-erjs": 2, "ervs-nojump": 3}
RNG = {"mt19937": 0, "philox": 1}

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
u16p = C.POINTER(C.c_uint16)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)


class OrcGraph(C.Structure):
    _fields_ = [("nv", C.c_uint32), ("ne", C.c_uint64), ("row", u64p), ("col", u32p),
                ("prop", f32p), ("label", u16p), ("nmax", f64p), ("nsum", f64p)]


class OrcModel(C.Structure):
    _fields_ = [("kind", C.c_int), ("weighted", C.c_int), ("a", C.c_double),
                ("b", C.c_double), ("gamma", C.c_double), ("schema", u16p),
                ("schema_len", C.c_uint32)]


class OrcOpts(C.Structure):
    _fields_ = [("mode", C.c_int), ("walk_length", C.c_uint32), ("seed", C.c_uint64),
                ("cap_per_degree", C.c_uint64), ("edge_cost_ratio", C.c_double),
                ("rng", C.c_int), ("qid_base", C.c_uint64), ("qids", C.c_void_p),
                ("erjs_handoff", C.c_double)]


class OrcStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "queries", "query_errors", "dead_ends", "steps", "select_ervs", "select_erjs",
        "trials", "weight_reads", "rng_draws", "erjs_fallbacks")] + [
        ("sel_by_deg", (C.c_uint64 * 2) * 33)]

    def as_dict(self) -> dict:
        d = {n: int(getattr(self, n)) for n, _ in self._fields_ if n != "sel_by_deg"}
        d["selection_by_degree"] = [(int(self.sel_by_deg[b][0]), int(self.sel_by_deg[b][1]))
                                    for b in range(33)]
        return d


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.POINTER(OrcGraph)
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_mt19937_64.argtypes = [C.c_uint64, C.c_uint64, u64p]
        L.orc_libm.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                               C.c_uint64]
        L.orc_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.orc_walker_draw.restype = C.c_uint64
        L.orc_walker_draw.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64]
        L.orc_graph_build.restype = P
        L.orc_graph_build.argtypes = [u32p, u32p, f32p, u16p, C.c_uint64, C.c_int, C.c_int,
                                      C.c_uint64]
        L.orc_graph_from_csr.restype = P
        L.orc_graph_from_csr.argtypes = [C.c_uint32, C.c_uint64, u64p, u32p, f32p, u16p]
        L.orc_graph_free.argtypes = [P]
        L.orc_has_edge.argtypes = [P, C.c_uint32, C.c_uint32]
        L.orc_gen_uniform.restype = P
        L.orc_gen_uniform.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_int]
        L.orc_gen_ba.restype = P
        L.orc_gen_ba.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_int]
        L.orc_synth_weights.argtypes = [P, C.c_int, C.c_double, C.c_double, C.c_double,
                                        C.c_uint64]
        L.orc_rmat_samples.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, u32p, u32p]
        L.orc_gen_rmat.restype = P
        L.orc_gen_rmat.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64]
        L.orc_gen_rmat_par.restype = P
        L.orc_gen_rmat_par.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_double,
                                       C.c_double, C.c_uint64, C.c_int]
        L.orc_synth_philox.argtypes = [P, C.c_int, C.c_double, C.c_double, C.c_double,
                                       C.c_uint64]
        L.orc_run.argtypes = [P, C.POINTER(OrcModel), C.POINTER(OrcOpts), u32p, C.c_uint64,
                              u32p, u32p, C.POINTER(OrcStats), C.c_int]
        L.orc_transition_probs.restype = C.c_int64
        L.orc_transition_probs.argtypes = [P, C.POINTER(OrcModel), C.c_uint32, C.c_uint32,
                                           C.c_uint32, f64p]
        L.orc_decide.argtypes = [P, C.POINTER(OrcModel), C.c_uint32, C.c_uint32, C.c_uint32,
                                 C.c_double, f64p, f64p]
        L.orc_weight.restype = C.c_double
        L.orc_weight.argtypes = [P, C.POINTER(OrcModel), C.c_uint32, C.c_uint32, C.c_uint32,
                                 C.c_uint64]
        L.orc_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref() -> C.CDLL:
    """The reference's own code (oracle/_ref).  Raises if it was never built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            raise FileNotFoundError(REF_PATH)
        R = C.CDLL(REF_PATH)
        vp = C.c_void_p
        R.ref_last_error.restype = C.c_char_p
        R.ref_graph_from_csr.restype = vp
        R.ref_graph_from_csr.argtypes = [C.c_uint32, C.c_uint64, u64p, u32p, f32p, u16p]
        R.ref_graph_gen.restype = vp
        R.ref_graph_gen.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int]
        R.ref_synth.argtypes = [vp, C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64]
        R.ref_graph_free.argtypes = [vp]
        R.ref_graph_dims.argtypes = [vp, u32p, u64p, C.POINTER(C.c_int)]
        R.ref_graph_copy.argtypes = [vp, u64p, u32p, f32p, u16p, f64p, f64p]
        run_args = [vp, C.POINTER(OrcModel), C.c_int, C.c_uint32, C.c_uint32, C.c_uint64,
                    C.c_uint64, C.c_double, u32p, C.c_uint64, u32p, u32p, C.POINTER(OrcStats),
                    f64p]
        R.ref_run.argtypes = run_args
        R.ref_run_philox.argtypes = run_args
        R.ref_profile_ratio.restype = C.c_double
        R.ref_profile_ratio.argtypes = [vp, C.POINTER(OrcModel), C.c_uint64]
        R.ref_set_dsl_source.argtypes = [C.c_char_p]
        R.ref_dsl_codegen.restype = C.c_long
        R.ref_dsl_codegen.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, u32p, u32p]
        R.ref_save_binary.argtypes = [vp, C.c_char_p]
        R.ref_load_binary.restype = vp
        R.ref_load_binary.argtypes = [C.c_char_p]
        _ref = R
    return _ref


def _ptr(a: np.ndarray | None, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def derive_seed(seed: int, stream: int) -> int:
    return int(lib().orc_derive_seed(seed & (2**64 - 1), stream & (2**64 - 1)))


@dataclass
class Model:
    """Builtin walk model (models.hpp:33-164); kind in MODEL_KINDS."""
    kind: str = "node2vec"
    weighted: bool = True
    a: float = 2.0
    b: float = 0.5
    gamma: float = 0.2
    schema: tuple = (0, 1, 2, 3, 4)
    _schema_arr: np.ndarray = field(default=None, repr=False)

    def c(self) -> OrcModel:
        self._schema_arr = np.asarray(self.schema, dtype=np.uint16)
        return OrcModel(MODEL_KINDS[self.kind], int(self.weighted), self.a, self.b, self.gamma,
                        _ptr(self._schema_arr, u16p), len(self.schema))

    def max_steps(self) -> int:
        return len(self.schema) if self.kind == "metapath" else 2**32 - 1


class Graph:
    """Oracle CSR (owned by liboracle)."""

    def __init__(self, ptr):
        if not ptr:
            raise RuntimeError(lib().orc_last_error().decode())
        self.ptr = ptr

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().orc_graph_free(self.ptr)
            self.ptr = None

    @property
    def nv(self) -> int:
        return int(self.ptr.contents.nv)

    @property
    def ne(self) -> int:
        return int(self.ptr.contents.ne)

    def arrays(self) -> dict:
        g = self.ptr.contents
        nv, ne = int(g.nv), int(g.ne)
        out = {
            "row": np.ctypeslib.as_array(g.row, (nv + 1,)).copy(),
            "col": np.ctypeslib.as_array(g.col, (ne,)).copy() if ne else np.zeros(0, np.uint32),
            "prop": np.ctypeslib.as_array(g.prop, (ne,)).copy() if ne else np.zeros(0, np.float32),
            "nmax": np.ctypeslib.as_array(g.nmax, (nv,)).copy(),
            "nsum": np.ctypeslib.as_array(g.nsum, (nv,)).copy(),
            "label": None,
        }
        if g.label and ne:
            out["label"] = np.ctypeslib.as_array(g.label, (ne,)).copy()
        return out

    @staticmethod
    def build(src, dst, prop=None, label=None, mirror=False, nv_hint=0) -> "Graph":
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        prop = None if prop is None else np.ascontiguousarray(prop, np.float32)
        label = None if label is None else np.ascontiguousarray(label, np.uint16)
        return Graph(lib().orc_graph_build(_ptr(src, u32p), _ptr(dst, u32p), _ptr(prop, f32p),
                                           _ptr(label, u16p), len(src), int(label is not None),
                                           int(mirror), nv_hint))

    @staticmethod
    def from_csr(row, col, prop, label=None) -> "Graph":
        row = np.ascontiguousarray(row, np.uint64)
        col = np.ascontiguousarray(col, np.uint32)
        prop = np.ascontiguousarray(prop, np.float32)
        label = None if label is None else np.ascontiguousarray(label, np.uint16)
        return Graph(lib().orc_graph_from_csr(len(row) - 1, len(col), _ptr(row, u64p),
                                              _ptr(col, u32p), _ptr(prop, f32p),
                                              _ptr(label, u16p)))

    @staticmethod
    def ba(n, deg, seed, mirror=True) -> "Graph":
        return Graph(lib().orc_gen_ba(n, deg, seed, int(mirror)))

    @staticmethod
    def uniform(n, deg, seed, mirror=True) -> "Graph":
        return Graph(lib().orc_gen_uniform(n, deg, seed, int(mirror)))

    @staticmethod
    def rmat(scale, edge_factor, seed) -> "Graph":
        return Graph(lib().orc_gen_rmat(scale, edge_factor, seed))

    @staticmethod
    def rmat_par(scale, edge_factor, seed, low=1.0, high=5.0, weight_seed=0, threads=None):
        threads = threads or os.cpu_count() or 1
        return Graph(lib().orc_gen_rmat_par(scale, edge_factor, seed, low, high, weight_seed,
                                            threads))

    def synth(self, kind: str, low=1.0, high=5.0, alpha=1.0, seed=0) -> "Graph":
        k = {"uniform": 0, "labels": 1, "pareto": 2, "degree": 3}[kind]
        if lib().orc_synth_weights(self.ptr, k, low, high, alpha, seed) != 0:
            raise RuntimeError(lib().orc_last_error().decode())
        return self

    def synth_philox(self, kind: str, low=1.0, high=5.0, alpha=1.0, seed=0) -> "Graph":
        k = {"uniform": 0, "labels": 1, "pareto": 2}[kind]
        if lib().orc_synth_philox(self.ptr, k, low, high, alpha, seed) != 0:
            raise RuntimeError(lib().orc_last_error().decode())
        return self

    def has_edge(self, v, u) -> bool:
        return bool(lib().orc_has_edge(self.ptr, v, u))


@dataclass
class RunResult:
    paths: np.ndarray      # nq x (L+1), INVALID padded
    lengths: np.ndarray    # nq
    stats: dict
    wall_ms: float = 0.0


def run(g: Graph, model: Model, queries, mode="adaptive", walk_length=80, seed=0,
        cap_per_degree=64, ratio=1.0, rng="philox", threads=1, keep_paths=True,
        qid_base=0, qids=None, erjs_handoff=0.0) -> RunResult:
    """Oracle run_queries (runtime.cpp:192-247).  qids: [nq] global walker
    ids (stream keys) of the queries, default qid_base + i."""
    q = np.ascontiguousarray(queries, np.uint32)
    qa = None if qids is None else np.ascontiguousarray(qids, np.uint64)
    if qa is not None and len(qa) != len(q):
        raise ValueError("qids must hold one id per query")
    paths = np.empty((len(q), walk_length + 1), np.uint32) if keep_paths else None
    lengths = np.empty(len(q), np.uint32)
    st = OrcStats()
    m = model.c()
    o = OrcOpts(MODES[mode], walk_length, seed, cap_per_degree, ratio, RNG[rng], qid_base,
                None if qa is None else qa.ctypes.data, erjs_handoff)
    import time
    t0 = time.perf_counter()
    rc = lib().orc_run(g.ptr, C.byref(m), C.byref(o), _ptr(q, u32p), len(q),
                       _ptr(paths, u32p), _ptr(lengths, u32p), C.byref(st), threads)
    t1 = time.perf_counter()
    if rc != 0:
        raise RuntimeError(lib().orc_last_error().decode())
    return RunResult(paths, lengths, st.as_dict(), (t1 - t0) * 1e3)


def transition_probs(g: Graph, model: Model, cur, prev=INVALID, step=0):
    row =np.ctypeslib.as_array(g.ptr.contents.row, (g.nv + 1,))
    d = int(row[cur + 1] - row[cur])
    out = np.zeros(max(d, 1), np.float64)
    m = model.c()
    r = lib().orc_transition_probs(g.ptr, C.byref(m), cur, prev, step, _ptr(out, f64p))
    if r < 0:
        raise RuntimeError(lib().orc_last_error().decode())
    return None if r == 0 else out[:d]


class RefGraph:
    """A dynwalk::Graph owned by the reference library."""

    def __init__(self, ptr):
        if not ptr:
            raise RuntimeError(ref().ref_last_error().decode())
        self.ptr = C.c_void_p(ptr)

    def __del__(self):
        if getattr(self, "ptr", None):
            ref().ref_graph_free(self.ptr)
            self.ptr = None

    @staticmethod
    def from_csr(row, col, prop, label=None) -> "RefGraph":
        row = np.ascontiguousarray(row, np.uint64)
        col = np.ascontiguousarray(col, np.uint32)
        prop = np.ascontiguousarray(prop, np.float32)
        label = None if label is None else np.ascontiguousarray(label, np.uint16)
        return RefGraph(ref().ref_graph_from_csr(len(row) - 1, len(col), _ptr(row, u64p),
                                                 _ptr(col, u32p), _ptr(prop, f32p),
                                                 _ptr(label, u16p)))

    @staticmethod
    def gen(kind: str, n, deg, seed, mirror=True) -> "RefGraph":
        return RefGraph(ref().ref_graph_gen({"uniform": 0, "ba": 1}[kind], n, deg, seed,
                                            int(mirror)))

    def synth(self, kind, low=1.0, high=5.0, alpha=1.0, seed=0) -> "RefGraph":
        k = {"uniform": 0, "labels": 1, "pareto": 2, "degree": 3}[kind]
        if ref().ref_synth(self.ptr, k, low, high, alpha, seed) != 0:
            raise RuntimeError(ref().ref_last_error().decode())
        return self

    def save_binary(self, path: str) -> None:
        """dynwalk::save_binary (graph.cpp:243-256): the DWG1 CSR cache."""
        if ref().ref_save_binary(self.ptr, path.encode()) != 0:
            raise RuntimeError(ref().ref_last_error().decode())

    @staticmethod
    def load_binary(path: str) -> "RefGraph":
        """dynwalk::load_binary (graph.cpp:258-291)."""
        return RefGraph(ref().ref_load_binary(path.encode()))

    def arrays(self) -> dict:
        nv, ne, hl = C.c_uint32(), C.c_uint64(), C.c_int()
        ref().ref_graph_dims(self.ptr, C.byref(nv), C.byref(ne), C.byref(hl))
        nv, ne = nv.value, ne.value
        out = {"row": np.empty(nv + 1, np.uint64), "col": np.empty(ne, np.uint32),
               "prop": np.empty(ne, np.float32), "nmax": np.empty(nv, np.float64),
               "nsum": np.empty(nv, np.float64),
               "label": np.empty(ne, np.uint16) if hl.value else None}
        ref().ref_graph_copy(self.ptr, _ptr(out["row"], u64p), _ptr(out["col"], u32p),
                             _ptr(out["prop"], f32p), _ptr(out["label"], u16p),
                             _ptr(out["nmax"], f64p), _ptr(out["nsum"], f64p))
        return out


def ref_run(g: RefGraph, model: Model, queries, mode="adaptive", walk_length=80, seed=0,
            cap_per_degree=64, ratio=1.0, rng="mt19937", workers=1,
            keep_paths=True) -> RunResult:
    """The reference's run_queries (rng='mt19937') or its sampler templates
    under the Philox walker stream (rng='philox')."""
    q = np.ascontiguousarray(queries, np.uint32)
    paths = np.empty((len(q), walk_length + 1), np.uint32) if keep_paths else None
    lengths = np.empty(len(q), np.uint32)
    st = OrcStats()
    wall = C.c_double()
    m = model.c()
    fn = ref().ref_run if rng == "mt19937" else ref().ref_run_philox
    rc = fn(g.ptr, C.byref(m), MODES[mode], walk_length, workers, seed, cap_per_degree, ratio,
            _ptr(q, u32p), len(q), _ptr(paths, u32p), _ptr(lengths, u32p), C.byref(st),
            C.byref(wall))
    if rc != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return RunResult(paths, lengths, st.as_dict(), wall.value)


def ref_profile_ratio(g: RefGraph, model: Model, seed: int) -> float:
    m = model.c()
    r = ref().ref_profile_ratio(g.ptr, C.byref(m), seed)
    if r < 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return r


def dsl_codegen(source: str):
    """The product's DSL -> CUDA model codegen (paper_2512_00705_b200/host/
    dsl_codegen.hpp) applied to the reference's parse/analysis of `source`.
    Returns (cuda_source, max_steps, flags)."""
    R = ref()
    ms, fl = C.c_uint32(), C.c_uint32()
    n = R.ref_dsl_codegen(source.encode(), None, 0, C.byref(ms), C.byref(fl))
    if n < 0:
        raise RuntimeError(R.ref_last_error().decode())
    buf = C.create_string_buffer(n + 1)
    R.ref_dsl_codegen(source.encode(), buf, n + 1, C.byref(ms), C.byref(fl))
    return buf.value.decode(), ms.value, fl.value


def set_dsl_source(source: str) -> None:
    """The program ModelDesc kind 4 ("dsl") parses on the reference side."""
    ref().ref_set_dsl_source(source.encode())
