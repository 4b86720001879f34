"""CPU: the host ImgQL front end builds the reference's task graphs.

Golden DAG dumps (tests/golden/reference_dags.json) come from the
reference's own parser + expander (TaskGraph::dump, task_graph.cpp:72-95).
Error cases follow proj/tests/test_frontend.cpp / test_task_graph.cpp.
"""
import json
import os

import numpy as np
import pytest

from paper_2010_07284_b200 import imgql as Q

HERE = os.path.dirname(os.path.abspath(__file__))
D = json.load(open(os.path.join(HERE, "golden", "reference_dags.json")))


@pytest.mark.parametrize("name", sorted(D["specs"]))
def test_dag_dump_matches_reference(name):
    assert Q.compile_text(D["specs"][name]).dump() == D["dumps"][name]


def test_segmentation_dag_counts():
    # test_task_graph.cpp:50-67: 10 nodes, one reach
    g = Q.compile_text(D["specs"]["segmentation"])
    assert g.node_count() == 10
    assert g.count_opcode("reach") == 1


def test_hash_consing_shares_subexpressions():
    g = Q.compile_text('load x = "m.png"\nsave "o.png" near(x) & !near(x)\n')
    assert g.count_opcode("near") == 1


def test_toposort_is_id_order():
    g = Q.compile_text(D["specs"]["c1"])
    assert g.toposort() == list(range(g.node_count()))
    for i, t in enumerate(g.nodes):
        assert all(d < i for d in t.deps)


@pytest.mark.parametrize("text,msg", [
    ('save "o.png" y\n', "unbound identifier 'y'"),
    ('let near(a) = a\n', "redefines a built-in"),
    ('let f(a) = f(a)\n', "used inside its own definition"),
    ('load x = "a.png"\nsave "o.png" near(x, x)\n', "expects 1 argument(s), got 2"),
    ('load x = "a.png"\nsave "o.png" x(1)\n', "is an image, not a function"),
    ('let f(a,b) = a\nsave "o.png" f(1)\n', "expects 2 argument(s), got 1"),
])
def test_expansion_errors(text, msg):
    with pytest.raises(Q.SpecError, match=msg.replace("(", r"\(").replace(")", r"\)")):
        Q.compile_text(text)


@pytest.mark.parametrize("text,msg", [
    ('let x = 1 +\n', "expected an expression"),
    ('save "" 1\n', "must not be empty"),
    ('let a = 1\nlet a = 2\n', "duplicate declaration"),
    ('let f(a, a) = a\n', "duplicate parameter"),
    ('print "x" 1 $ 2\n', "unexpected character"),
    ('load x = "unterminated\n', "unterminated string literal"),
])
def test_parse_errors(text, msg):
    with pytest.raises(Q.SpecError, match=msg):
        Q.compile_text(text)


def test_precedence_and_associativity():
    g = Q.compile_text('print "p" 1 - 2 - 3 * 4 / 2\n')
    # ((1 - 2) - ((3 * 4) / 2)); the second `2` is hash-consed onto node 1
    ops = [t.opcode for t in g.nodes]
    assert ops == ["const", "const", "-", "const", "const", "*", "/", "-", "print"]
    assert g.nodes[6].deps == (5, 1) and g.nodes[7].deps == (2, 6)


def test_maxvol_is_a_builtin_here():
    g = Q.compile_text('load x = "a.png"\nsave "o.png" maxvol(x > . 1)\n'.replace("> .", ">."))
    assert g.count_opcode("maxvol") == 1


def test_payload_text_matches_to_chars():
    assert Q.payload_text(62258.0) == "62258"
    assert Q.payload_text(0.5) == "0.5"
    assert Q.payload_text(1e300) == "1e+300"
    assert Q.payload_text(1e-7) == "1e-07"
    assert Q.payload_text("a.png") == '"a.png"'


def test_corrected_spiral_is_one_long_component():
    # synth::generate(Spiral) with the Bresenham fix: deterministic, a single
    # 8-connected curve (the reference generator never terminates)
    import oracle as O
    from paper_2010_07284_b200 import synth as S
    a = S.spiral(300, 260, 5)
    assert np.array_equal(a, S.spiral(300, 260, 5))
    m = (a > 0).astype(np.uint8)
    assert m.sum() > 1500
    assert len(np.unique(O.flood_fill_label(m))) == 2  # background + one component
