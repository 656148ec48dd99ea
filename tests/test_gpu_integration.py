"""The reference-side binding of INTEGRATION.md §2, executed verbatim.

The ctypes stub a maintainer of the reference would add (``cntgw/_b200.py``)
is extracted from INTEGRATION.md and run against the in-tree
``libcntgw_b200.so`` on the C1 final plan: its ``softmin_sq_euclidean`` must
reproduce the reference ``_softmin`` (sinkhorn.py:166-176; the oracle,
pinned to the reference by tests/test_oracle.py) on the same inputs.
"""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu


def _stub_source():
    text = open(os.path.join(ROOT, "INTEGRATION.md"), encoding="utf-8").read()
    section = text[text.index("## 2. Binding the C ABI"):]
    return re.search(r"```python\n(.*?)```", section, re.S).group(1)


def test_integration_stub_matches_reference_softmin(cuda, monkeypatch):
    from oracle import cntgw_oracle as O

    monkeypatch.setenv("CNTGW_B200_LIB",
                       os.path.join(ROOT, "paper_2602_06658_b200", "libcntgw_b200.so"))
    ns = {}
    exec(compile(_stub_source(), "INTEGRATION.md", "exec"), ns)  # noqa: S102
    gold = golden("c1_solve")
    x, z, eps = gold["xbar"], gold["zbar"], float(gold["eps_eff"])
    log_b = np.log(gold["b"])
    got = ns["softmin_sq_euclidean"](x, z, log_b, gold["g"], eps)
    want = O.softmin(O.SqEuclid(x, z), log_b, gold["g"], eps)
    # the fp64 path forms exponents in fp64 and sums 2^(offset) on MUFU.EX2
    # with the offset (32-48 log2 units) truncated to fp32: <= ~3e-6 log2
    # units per LSE, i.e. an absolute error of a few 1e-6 eps
    tol = 1e-7 * np.abs(want).max() + 4e-6 * eps
    assert np.abs(got - want).max() <= tol
    # the g side through the same stub (transposed provider)
    got_g = ns["softmin_sq_euclidean"](z, x, np.log(gold["a"]), gold["f"], eps)
    want_g = O.softmin(O.SqEuclid(z, x), np.log(gold["a"]), gold["f"], eps)
    assert np.abs(got_g - want_g).max() <= 1e-7 * np.abs(want_g).max() + 4e-6 * eps
