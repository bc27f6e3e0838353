"""The native chain-file loader (csrc/host/chain_file.cpp, load_chain_json of
proj/include/ooc/chain_file.hpp:22-23) on CPU: the reference's format ("loops"), this repo's
"ops" extension, fills, named stencils, and the reference's validation errors
(proj/src/chain_file.cpp:12-52, 118-140)."""
import json

import pytest

import paper_1709_02125_b200 as B

BASE = {
    "datasets": [{"name": "u", "core": {"lo": [0, 0], "hi": [16, 12]}, "halo": 1, "fill": "(+ 1 (* 0.5 i))"},
                 {"name": "t", "core": {"lo": [0, 0], "hi": [16, 12]}, "halo": [1, 1]}],
    "stencils": [{"name": "s5", "offsets": [[0, 0], [-1, 0], [1, 0], [0, -1], [0, 1]]}],
    "loops": [{"range": {"lo": [1, 1], "hi": [15, 11]},
               "args": [{"dataset": "u", "stencil": "s5", "mode": "READ"},
                        {"dataset": "t", "stencil": "point", "mode": "WRITE"}],
               "kernel": {"writes": {"1": "(* 0.25 (+ (+ (r 0 -1 0) (r 0 1 0)) (+ (r 0 0 -1) (r 0 0 1))))"},
                          "reduction": {"op": "SUM", "expr": "(r 0 0 0)", "name": "usum"}}}],
}


def _rt():
    return B.Runtime("plan_only", record=True, tiles=1)


def test_reference_format_loads_and_plans():
    rt = B.load_program(_rt(), BASE)
    assert rt.num_datasets == 2
    assert rt.find("u") == 0 and rt.find("t") == 1
    assert rt.flush_log() == [[0, "REDUCTION_FETCH", 1]]  # a reducing loop flushes after itself
    u = rt.host(0)
    assert u[1, 1] == 1.0 and u[2, 1] == 1.5  # fill (+ 1 (* 0.5 i)) at i = 0, 1 (halo row first)


def test_ops_extension_interleaves_flushes():
    prog = dict(BASE)
    loop = dict(BASE["loops"][0])
    loop["kernel"] = {"writes": loop["kernel"]["writes"]}
    prog = {k: v for k, v in BASE.items() if k != "loops"}
    prog["ops"] = [dict(loop, op="loop"), {"op": "flush"}, {"op": "cyclic", "on": True}, dict(loop, op="loop"),
                   {"op": "finish"}]
    rt = B.load_program(_rt(), json.dumps(prog))
    assert [f[2] for f in rt.flush_log()] == [1, 1]


@pytest.mark.parametrize("mutate,msg", [
    (lambda p: p["loops"][0]["args"][0].update(dataset="nope"), "unknown dataset 'nope'"),
    (lambda p: p["loops"][0]["args"][0].update(stencil="s9"), "unknown stencil 's9'"),
    (lambda p: p["loops"][0]["args"][0].update(mode="RW"), "unknown access mode 'RW'"),
    (lambda p: p["loops"][0]["kernel"]["reduction"].update(op="AVG"), "unknown reduction op 'AVG'"),
    (lambda p: p["datasets"][0].update(halo=[1, 1, 1]), "halo array rank"),
    (lambda p: p["datasets"][0].update(fill=[1.0]), "fill must be a number or an expression"),
    (lambda p: p["datasets"][0]["core"].update(hi=[16]), "matching rank"),
])
def test_reference_validation_errors(mutate, msg):
    prog = json.loads(json.dumps(BASE))
    mutate(prog)
    with pytest.raises(B.ValidationError, match=msg):
        B.load_program(_rt(), prog)


def test_malformed_json_is_a_validation_error():
    with pytest.raises(B.ValidationError, match="JSON parse error"):
        B.load_program(_rt(), '{"datasets": [')
