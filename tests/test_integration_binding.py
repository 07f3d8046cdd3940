"""INTEGRATION.md's reference-side ctypes binding (the stub a maintainer adds
as qdot/_b200.py) is executed as written: on CPU its structures must match
the C ABI and the symbol must resolve; on the GPU it must return the same
value and bins as the package's qdot()."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_binding():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("### The reference-side binding"):]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    assert 'ctypes.CDLL("libqdot_b200.so")' in code
    code = code.replace('ctypes.CDLL("libqdot_b200.so")', f'ctypes.CDLL({_lib.lib_path()!r})')
    ns = {}
    exec(compile(code, "INTEGRATION.md:qdot/_b200.py", "exec"), ns)
    return ns


def test_binding_structs_match_the_c_abi():
    if not os.path.exists(_lib.lib_path()):
        pytest.skip("library not built")
    ns = load_binding()
    assert ctypes.sizeof(ns["_Bin"]) == ctypes.sizeof(_lib.QdotBin) == 56
    assert ctypes.sizeof(ns["_Res"]) == ctypes.sizeof(_lib.QdotResult)
    assert ctypes.sizeof(ns["_Cfg"]) == ctypes.sizeof(_lib.QdotConfig)
    for a, b in ((ns["_Bin"], _lib.QdotBin), (ns["_Res"], _lib.QdotResult), (ns["_Cfg"], _lib.QdotConfig)):
        assert [f[0] for f in a._fields_] == [f[0] for f in b._fields_]
        for (name, _), (_, _) in zip(a._fields_, b._fields_):
            assert getattr(a, name).offset == getattr(b, name).offset, name
    assert hasattr(ns["_lib"], "qdot_b200_dot_host")


@pytest.mark.gpu
@pytest.mark.parametrize("strategy,split", [("exact", "none"), ("ranged:3", "per-bin"), ("split:4", "none")])
def test_binding_matches_qdot(strategy, split):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ns = load_binding()
    rng = np.random.default_rng(5)
    x = rng.standard_normal(300001)
    y = rng.standard_normal(300001)
    cfg = Q.ToleranceConfig(1e-7, Q.SplitMode(split))
    st = Q.parse_strategy(strategy)
    r, bins = ns["b200_qdot"](x, y, cfg, st)
    rep = Q.qdot(x, y, cfg, strategy=st)
    assert r.value == rep.value
    assert [(b.lower, b.upper, b.cardinality, b.score, b.precision) for b in bins] == \
        [(b.lower, b.upper, b.cardinality, b.score, b.precision.code) for b in rep.params.bins]
    with pytest.raises(ValueError):
        ns["b200_qdot"](np.array([1.0, np.inf]), np.ones(2), cfg, st)
