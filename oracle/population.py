"""Reference (CPU) generic Population -- TEST INFRASTRUCTURE ONLY.

The plain definition of SPEC's columnar-core semantics (Sec. 3.1.2,
Listing 1; Sec. 3.3): numpy columns, a tombstone alive mask,
sequential never-reused ids, order-preserving compaction, and postfix
expression programs evaluated column-wise in float64 with the stored dtype's
conversion (truncation toward zero for integer columns, round-to-nearest for
float32).  RAND draws come from this oracle's own Philox (oracle.lane32).
"""
import numpy as np

from . import lane32

NP = {"i32": np.int32, "i64": np.int64, "f32": np.float32, "f64": np.float64, "u8": np.uint8}


class PopulationRef:
    def __init__(self, schema, seed=0):
        self.names = list(schema)
        self.dt = {k: NP[v] for k, v in schema.items()}
        self.cols = {k: np.zeros(0, self.dt[k]) for k in self.names}
        self.alive = np.zeros(0, bool)
        self.ids = np.zeros(0, np.int64)
        self.next_id = 0
        self.seed = seed
        self.step = 0

    def add_agents(self, n, **defaults):
        for k in self.names:
            self.cols[k] = np.concatenate([self.cols[k], np.full(n, defaults.get(k, 0), self.dt[k])])
        ids = np.arange(self.next_id, self.next_id + n, dtype=np.int64)
        self.ids = np.concatenate([self.ids, ids])
        self.alive = np.concatenate([self.alive, np.ones(n, bool)])
        self.next_id += n
        return ids

    def _rows(self, ids):
        rows = []
        for i in ids:
            r = np.nonzero(self.ids == i)[0]
            if r.size == 0 or not self.alive[r[0]]:
                raise ValueError(f"unknown or dead id {i}")
            rows.append(r[0])
        return np.array(rows, np.int64)

    def remove_agents(self, ids):
        if len(set(ids)) != len(ids):
            raise ValueError("duplicate id")
        self.alive[self._rows(ids)] = False

    def compact(self):
        keep = self.alive
        for k in self.names:
            self.cols[k] = self.cols[k][keep]
        self.ids = self.ids[keep]
        self.alive = self.alive[keep]

    def eval(self, prog):
        st = []
        n = self.ids.size
        for op, arg, val in prog:
            if op == "CONST":
                st.append(np.full(n, val, np.float64))
            elif op == "COL":
                st.append(self.cols[arg].astype(np.float64))
            elif op == "ID":
                st.append(self.ids.astype(np.float64))
            elif op == "STEP":
                st.append(np.full(n, float(self.step)))
            elif op == "RAND":
                st.append(np.array([((lane32(self.seed, arg, int(i), self.step) >> 8) * 2.0 ** -24)
                                    for i in self.ids], np.float64))
            elif op in ("NEG", "ABS", "FLOOR", "SQRT", "NOT"):
                a = st.pop()
                np.seterr(invalid="ignore")
                st.append({"NEG": lambda x: -x, "ABS": np.abs, "FLOOR": np.floor,
                           "SQRT": np.sqrt,
                           "NOT": lambda x: (x == 0).astype(np.float64)}[op](a))
            elif op == "SELECT":
                b, a, c = st.pop(), st.pop(), st.pop()
                st.append(np.where(c != 0, a, b))
            else:
                b, a = st.pop(), st.pop()
                f = {"ADD": np.add, "SUB": np.subtract, "MUL": np.multiply, "DIV": np.divide,
                     "MIN": np.fmin, "MAX": np.fmax, "LT": np.less, "LE": np.less_equal,
                     "GT": np.greater, "GE": np.greater_equal, "EQ": np.equal, "NE": np.not_equal,
                     "AND": lambda x, y: (x != 0) & (y != 0), "OR": lambda x, y: (x != 0) | (y != 0)}[op]
                with np.errstate(all="ignore"):
                    st.append(np.asarray(f(a, b), np.float64))
        assert len(st) == 1
        return st[0]

    def eval_tree(self, t):
        """The plain definition of an expression given as a tuple tree,
        independent of the product's Expr lowering: ("col", name), ("const", v),
        ("id",), ("step",), ("rand", tag), (unary, a) for neg / abs / floor /
        sqrt / not, ("select", c, a, b), (binary, a, b) for add / sub / mul / div
        / min / max / lt / le / gt / ge / eq / ne / and / or -- every value a
        float64 column, comparisons 1.0 / 0.0, min / max ignoring NaN (fmin /
        fmax), as SPEC's float64 evaluation."""
        n = self.ids.size
        k = t[0]
        if k == "col":
            return self.cols[t[1]].astype(np.float64)
        if k == "const":
            return np.full(n, float(t[1]))
        if k == "id":
            return self.ids.astype(np.float64)
        if k == "step":
            return np.full(n, float(self.step))
        if k == "rand":
            return np.array([((lane32(self.seed, t[1], int(i), self.step) >> 8) * 2.0 ** -24) for i in self.ids],
                            np.float64)
        with np.errstate(all="ignore"):
            if k == "select":
                c, a, b = (self.eval_tree(x) for x in t[1:])
                return np.where(c != 0, a, b)
            if len(t) == 2:
                a = self.eval_tree(t[1])
                return {"neg": lambda x: -x, "abs": np.abs, "floor": np.floor, "sqrt": np.sqrt,
                        "not": lambda x: (x == 0).astype(np.float64)}[k](a)
            a, b = self.eval_tree(t[1]), self.eval_tree(t[2])
            f = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "div": np.divide, "min": np.fmin,
                 "max": np.fmax, "lt": np.less, "le": np.less_equal, "gt": np.greater, "ge": np.greater_equal,
                 "eq": np.equal, "ne": np.not_equal, "and": lambda x, y: (x != 0) & (y != 0),
                 "or": lambda x, y: (x != 0) | (y != 0)}[k]
            return np.asarray(f(a, b), np.float64)

    def _value(self, e):
        return self.eval_tree(e) if isinstance(e, tuple) else self.eval(e)

    def update(self, target, prog, where=None):
        """prog / where: a postfix program (list) or an expression tree (tuple)."""
        sel = self.alive.copy()
        if where:
            sel &= self._value(where) != 0
        with np.errstate(all="ignore"):
            v = self._value(prog)
        self.cols[target] = self.cols[target].copy()
        self.cols[target][sel] = v[sel].astype(self.dt[target])
        return int(sel.sum())

    def aggregate(self, kind, prog=None, where=None):
        sel = self.alive.copy()
        if where:
            sel &= self._value(where) != 0
        if kind == "count":
            return float(sel.sum())
        v = self._value(prog)[sel]
        if kind == "sum":
            return float(v.sum())
        if v.size == 0:
            raise ValueError("empty selection")
        return float({"mean": np.mean, "min": np.min, "max": np.max}[kind](v))

    def column(self, name):
        return (self.ids if name == "id" else self.cols[name])[self.alive]

    def batch_set(self, name, ids, values):
        rows = self._rows(ids)  # validate everything first
        c = self.cols[name].copy()
        for r, v in zip(rows, values):  # staging order: the last write wins
            c[r] = np.asarray(v, np.float64).astype(self.dt[name])
        self.cols[name] = c
