"""Generic device Population (NEXT-4): the paper's columnar API over the C ABI.

    pop = Population({"wealth": "i64", "state": "u8"})
    ids = pop.add_agents(3, wealth=1)
    pop.update("wealth", col("wealth") + 10)          # PAPER.md Listing 1
    pop.update("wealth", col("wealth") - 5, where=col("wealth") >= 5)
    pop.aggregate("sum", col("wealth"))

Expressions are built with Python operators and compiled to the ABI's postfix
program (amber_instr); every evaluation runs in libamber.so's kernels.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .capi import check
from .model import make_runtime

DTYPES = {"i32": capi.AMBER_I32, "i64": capi.AMBER_I64, "f32": capi.AMBER_F32, "f64": capi.AMBER_F64,
          "u8": capi.AMBER_U8}
NP = {"i32": np.int32, "i64": np.int64, "f32": np.float32, "f64": np.float64, "u8": np.uint8}
OP = dict(CONST=0, COL=1, ID=2, STEP=3, ADD=10, SUB=11, MUL=12, DIV=13, MIN=14, MAX=15, NEG=20, ABS=21,
          FLOOR=22, SQRT=23, LT=30, LE=31, GT=32, GE=33, EQ=34, NE=35, AND=40, OR=41, NOT=42, SELECT=50,
          RAND=60)
AGG = {"sum": 0, "mean": 1, "min": 2, "max": 3, "count": 4}


class Expr:
    """A postfix program over columns (symbolic names until compiled)."""

    def __init__(self, prog):
        self.prog = prog  # list of (op name, arg, value)

    @staticmethod
    def of(v):
        return v if isinstance(v, Expr) else Expr([("CONST", 0, float(v))])

    def _bin(self, op, o, swap=False):
        a, b = (Expr.of(o), self) if swap else (self, Expr.of(o))
        return Expr(a.prog + b.prog + [(op, 0, 0.0)])

    def __add__(self, o): return self._bin("ADD", o)
    def __radd__(self, o): return self._bin("ADD", o, True)
    def __sub__(self, o): return self._bin("SUB", o)
    def __rsub__(self, o): return self._bin("SUB", o, True)
    def __mul__(self, o): return self._bin("MUL", o)
    def __rmul__(self, o): return self._bin("MUL", o, True)
    def __truediv__(self, o): return self._bin("DIV", o)
    def __rtruediv__(self, o): return self._bin("DIV", o, True)
    def __lt__(self, o): return self._bin("LT", o)
    def __le__(self, o): return self._bin("LE", o)
    def __gt__(self, o): return self._bin("GT", o)
    def __ge__(self, o): return self._bin("GE", o)
    def __eq__(self, o): return self._bin("EQ", o)  # noqa: D105 (expression, not identity)
    def __ne__(self, o): return self._bin("NE", o)
    def __and__(self, o): return self._bin("AND", o)
    def __or__(self, o): return self._bin("OR", o)
    def __neg__(self): return Expr(self.prog + [("NEG", 0, 0.0)])
    def __invert__(self): return Expr(self.prog + [("NOT", 0, 0.0)])
    __hash__ = None

    def min(self, o): return self._bin("MIN", o)
    def max(self, o): return self._bin("MAX", o)
    def abs(self): return Expr(self.prog + [("ABS", 0, 0.0)])
    def floor(self): return Expr(self.prog + [("FLOOR", 0, 0.0)])
    def sqrt(self): return Expr(self.prog + [("SQRT", 0, 0.0)])

    def where(self, a, b):
        """self != 0 ? a : b"""
        return Expr(self.prog + Expr.of(a).prog + Expr.of(b).prog + [("SELECT", 0, 0.0)])


def col(name: str) -> Expr:
    return Expr([("COL", name, 0.0)])


def lit(v) -> Expr:
    return Expr.of(v)


def agent_id() -> Expr:
    return Expr([("ID", 0, 0.0)])


def step_index() -> Expr:
    return Expr([("STEP", 0, 0.0)])


def rand(tag: int) -> Expr:
    """Uniform [0,1) Philox draw keyed on (population seed, tag, agent id, step)."""
    return Expr([("RAND", int(tag), 0.0)])


class Population:
    def __init__(self, schema: dict, capacity: int = 16, seed: int = 0, device=0, stream=None,
                 torch_alloc=True):
        self.lib = capi.lib()
        self.names = list(schema)
        self.dtypes = [schema[k] for k in self.names]
        specs = (capi.amber_column_spec * len(self.names))()
        self._keep = [k.encode() for k in self.names]
        for i, (k, d) in enumerate(zip(self._keep, self.dtypes)):
            specs[i].name = k
            specs[i].dtype = DTYPES[d]
        self.rt = make_runtime(device, stream, torch_alloc)
        self.stream = self.rt._keep[0]
        h = C.c_void_p()
        check(self.lib.amber_population_create(specs, len(self.names), int(capacity), int(seed),
                                               C.byref(self.rt), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            check(self.lib.amber_population_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- agents
    def add_agents(self, n: int, **defaults):
        d = (C.c_double * max(len(self.names), 1))(*[float(defaults.get(k, 0.0)) for k in self.names])
        first = C.c_int64()
        check(self.lib.amber_population_add_agents(self.h, int(n), d, C.byref(first)))
        return np.arange(first.value, first.value + n, dtype=np.int64)

    def remove_agents(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        check(self.lib.amber_population_remove_agents(self.h, ids.ctypes.data_as(C.POINTER(C.c_int64)),
                                                      ids.size))

    def compact(self):
        check(self.lib.amber_population_compact(self.h))

    def size(self):
        live, rows = C.c_int64(), C.c_int64()
        check(self.lib.amber_population_size(self.h, C.byref(live), C.byref(rows)))
        return live.value, rows.value

    # -- expressions
    def _compile(self, e):
        if e is None:
            return None, 0
        e = Expr.of(e)
        arr = (capi.amber_instr * len(e.prog))()
        for i, (op, arg, val) in enumerate(e.prog):
            arr[i].op = OP[op]
            arr[i].arg = self.names.index(arg) if op == "COL" else int(arg)
            arr[i].value = float(val)
        return arr, len(e.prog)

    def update(self, target: str, expr, where=None, count: bool = True):
        """Returns the number of rows updated; count=False enqueues asynchronously (None)."""
        pe, ne = self._compile(expr)
        pw, nw = self._compile(where)
        k = C.c_int64()
        check(self.lib.amber_population_update(self.h, target.encode(), pe, ne, pw, nw,
                                               C.byref(k) if count else None))
        return k.value if count else None

    def update_paths(self):
        """(jit, interpreted) general-program update counts (amber_population_update_paths)."""
        j, i = C.c_int64(), C.c_int64()
        check(self.lib.amber_population_update_paths(self.h, C.byref(j), C.byref(i)))
        return j.value, i.value

    def synchronize(self):
        check(self.lib.amber_population_synchronize(self.h))

    def aggregate(self, kind: str, expr=None, where=None) -> float:
        pe, ne = self._compile(expr)
        pw, nw = self._compile(where)
        out = C.c_double()
        check(self.lib.amber_population_aggregate(self.h, AGG[kind], pe, ne, pw, nw, C.byref(out)))
        return out.value

    def column(self, name: str):
        live, _ = self.size()
        dt = np.int64 if name == "id" else NP[self.dtypes[self.names.index(name)]]
        out = np.empty(max(live, 1), dtype=dt)
        check(self.lib.amber_population_read_column(self.h, name.encode(), out.ctypes.data_as(C.c_void_p),
                                                    out.nbytes, 0))
        return out[:live]

    def batch_set(self, name: str, ids, values):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        vals = np.ascontiguousarray(values, dtype=np.float64)
        check(self.lib.amber_population_batch_set(self.h, name.encode(),
                                                  ids.ctypes.data_as(C.POINTER(C.c_int64)),
                                                  vals.ctypes.data_as(C.POINTER(C.c_double)), ids.size))

    def set_step(self, t: int):
        check(self.lib.amber_population_set_step(self.h, int(t)))
