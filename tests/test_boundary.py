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


def test_plan_rejects_non_shrinking_chain():
    """eps2 close to 1: the block chain would not shrink (s >= span; P:281 needs s_{i+1} < s_i):
    XC_ENUMERIC from the product's planner and ArithmeticError from the oracle's, no endless loop."""
    from paper_2004_11610_b200 import xc
    with pytest.raises(xc.XcError, match="XC_ENUMERIC"):
        xc.plan_chain(xc.XC_JACOBI, 65536, 1e-12, 0.9)
    with pytest.raises(ArithmeticError):
        O.make_plan(O.Kind(O.KIND_JACOBI), 65536, 1e-12, eps2=0.9)


def test_bench_multi_gpu_launch_plan():
    """bench.py --gpus N without a launcher re-launches itself as N ranks (torch.distributed.run on
    127.0.0.1); under the launcher the ranks split the config's global batch (strong scaling)."""
    from paper_2004_11610_b200.shard import rank_columns, relaunch_cmd, world_from
    assert world_from({}, 1) == (1, 0, 0, False)
    assert world_from({}, 2) == (1, 0, 0, True)
    assert world_from({"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"}, 2) == (2, 1, 1, False)
    assert world_from({"WORLD_SIZE": "4", "RANK": "3", "LOCAL_RANK": "3"}, 1) == (4, 3, 3, False)
    with pytest.raises(ValueError):
        world_from({"WORLD_SIZE": "2"}, 8)
    cmd = relaunch_cmd("bench.py", ["--gpus", "2", "--steps", "3"], 2, 29500)
    assert "--nproc-per-node=2" in cmd and "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "2", "--steps", "3"]
    B = I.CONFIGS["c5"].B
    for G in (1, 2, 4, 8):
        sh = [rank_columns(B, g, G) for g in range(G)]
        assert sum(s.stop - s.start for s in sh) == B == 4096 and sh[0].start == 0 and sh[-1].stop == B
        assert all(sh[g].stop == sh[g + 1].start for g in range(G - 1))
        assert rank_columns(B, G - 1, G, strong=False) == slice(0, B)
