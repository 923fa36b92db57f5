import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def csr_from_dense(a, p):
    """Host CSR (gbla_gen.CSR) from a dense integer matrix; zeros dropped."""
    from gbla_gen import CSR
    a = np.asarray(a, dtype=np.int64) % p
    m, n = a.shape
    rp = [0]
    cols, vals = [], []
    for i in range(m):
        nz = np.nonzero(a[i])[0]
        cols.extend(nz.tolist())
        vals.extend(a[i, nz].tolist())
        rp.append(len(cols))
    return CSR(m=m, n=n, p=p, row_ptr=np.array(rp, np.uint64), col=np.array(cols, np.uint32),
               val=np.array(vals, np.uint16))


@pytest.fixture(scope="session")
def c0_matrix():
    import gbla_gen
    return gbla_gen.f4_matrix("c0")


@pytest.fixture(scope="session")
def c0_oracle(c0_matrix):
    import oracle
    return oracle.reduce(c0_matrix, want_x=True)
