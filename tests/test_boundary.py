"""CPU checks of the C-ABI boundary: libxc.so loads and exports every symbol that
include/xc.h declares; the host-only planner equals the oracle's plan."""
import os
import re

import pytest

import oracle as O
from paper_2004_11610_b200 import inputs as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "xc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(xc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2004_11610_b200 import xc
    lib = xc.load()
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(xc.EXPORTS)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_host_plan_equals_oracle(cfg):
    """zeta, block chain and tail of the product's planner (host C++) = the oracle's (Python)."""
    from paper_2004_11610_b200 import xc
    c = I.CONFIGS[cfg]
    z, blocks, tail = xc.plan_chain(c.kind, c.N, c.eps)
    p = O.make_plan(O.Kind(c.kind, c.alpha, c.beta), c.N, c.eps)
    assert abs(z - p.zeta) <= 1e-12 * p.zeta
    assert blocks == [(b.L, b.m_off, b.keep_lo, b.keep_hi) for b in p.blocks]
    assert tail == p.tail


def test_plan_rejects_bad_eps():
    from paper_2004_11610_b200 import xc
    with pytest.raises(xc.XcError, match="XC_EINVAL"):
        xc.plan_chain(xc.XC_JACOBI, 512, 0.5, 0.1)
    with pytest.raises(xc.XcError, match="XC_EINVAL"):
        xc.plan_chain(xc.XC_JACOBI, 1, 1e-12)
