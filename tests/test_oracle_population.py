"""Pins for the reference Population (SPEC columnar-core examples; PAPER.md
Listing 1).  Every expected value is a worked example printed in SPEC.md or a
closed form, not a re-evaluation by the reference itself."""
import numpy as np
import pytest

from oracle.population import PopulationRef


# expressions as plain tuple trees (oracle.population.eval_tree): the pins do
# not go through the product's Expr lowering
def col(name):
    return ("col", name)


def add(a, v):
    return ("add", a, ("const", v))


def sub(a, v):
    return ("sub", a, ("const", v))


def cmp(op, a, v):
    return (op, a, ("const", v))


def test_listing1_increment():
    p = PopulationRef({"wealth": "i64"})
    assert p.add_agents(3, wealth=1).tolist() == [0, 1, 2]  # SPEC add_agents example
    p.update("wealth", add(col("wealth"), 10))  # PAPER.md Listing 1
    assert p.column("wealth").tolist() == [11, 11, 11]


def test_update_where_example():
    p = PopulationRef({"wealth": "i64"})
    p.add_agents(3)
    p.cols["wealth"][:] = [0, 5, 9]
    n = p.update("wealth", sub(col("wealth"), 5), cmp("ge", col("wealth"), 5))
    assert p.column("wealth").tolist() == [0, 0, 4] and n == 2
    assert p.update("wealth", add(col("wealth"), 1), cmp("gt", col("wealth"), 100)) == 0


def test_aggregate_examples():
    p = PopulationRef({"wealth": "i64"})
    p.add_agents(3)
    p.cols["wealth"][:] = [1, 2, 3]
    w = col("wealth")
    assert (p.aggregate("sum", w), p.aggregate("mean", w), p.aggregate("min", w), p.aggregate("max", w)) == \
        (6, 2.0, 1, 3)
    p.remove_agents([1])
    assert p.aggregate("sum", w) == 4 and p.aggregate("count") == 2
    q = PopulationRef({"x": "f64"})
    q.add_agents(5)
    q.remove_agents([0, 3])
    assert q.aggregate("count") == 3
    q.remove_agents([1, 2, 4])
    assert q.aggregate("sum", col("x")) == 0.0
    with pytest.raises(ValueError):
        q.aggregate("mean", col("x"))


def test_ids_never_reused_and_compact():
    p = PopulationRef({"v": "i32"})
    p.add_agents(3, v=7)
    p.remove_agents([1])
    assert p.add_agents(1).tolist() == [3]  # never 1
    with pytest.raises(ValueError):
        p.remove_agents([1])  # already dead
    p.compact()
    assert p.ids.tolist() == [0, 2, 3] and p.column("v").tolist() == [7, 7, 0]


def test_batch_atomic_last_wins():
    p = PopulationRef({"wealth": "i64"})
    p.add_agents(3)
    p.batch_set("wealth", [0, 1], [9, 4])  # SPEC begin/apply example
    assert p.column("wealth").tolist() == [9, 4, 0]
    with pytest.raises(ValueError):
        p.batch_set("wealth", [2, 99], [5, 5])
    assert p.column("wealth").tolist() == [9, 4, 0]  # nothing applied
    p.batch_set("wealth", [2, 2], [1, 8])
    assert p.column("wealth")[2] == 8


def test_dtype_conversion_rules():
    p = PopulationRef({"i": "i32", "f": "f32"})
    p.add_agents(2)
    p.update("i", sub(col("i"), 2.7))  # truncation toward zero
    p.update("f", add(col("f"), 0.1))  # round to nearest float32
    assert p.column("i").tolist() == [-2, -2]
    assert p.column("f")[0] == np.float32(0.1)
