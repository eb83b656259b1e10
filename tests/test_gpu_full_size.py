"""Full-size parity on all five BASELINE configs: every row of the sm_100a
engine (through the C-ABI) against the unmodified reference kernel
(oracle/_ref, compiled from /root/reference/proj/src by oracle/Makefile) run
on all host cores in the same process.

* C1-C4 at BASELINE size: every task, every field (score, h_ext, v_ext,
  cells, delta_w, status, spread) and every seed score.
* C5 at BASELINE size (2,000,000 extensions, 2.43e11 cells): every task as
  well; the reference takes ~2 minutes of 16 host cores for it.

The reference batch is the loop of proj/src/pipeline.cpp:103-136 (split_lr,
checked seed score, xdrop_extend per side, align.cpp:37-155), fed longest
first only to balance its threads; results land at their task index.
When oracle/_ref is missing the C restatement (oracle/liboracle.so, pinned
against the reference by tests/test_oracle.py) is the checker instead."""
import os
import time

import numpy as np
import pytest

from helpers import blosum62, oracle_scheme, result_rows_equal

pytestmark = pytest.mark.gpu


def _host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


@pytest.fixture(scope="module")
def xb():
    import paper_2304_08662_b200 as xb
    assert xb.capi.lib().xb_device_count() > 0, "no CUDA device: the engine has no CPU fallback"
    return xb


def _checker(ds):
    """(name, run(tasks) -> (rows, seed_scores)) for the reference, or the
    pinned C oracle when the reference library is absent."""
    from oracle_py import REF_SO, Oracle, Ref
    threads = _host_threads()
    ln = np.diff(ds.offsets)
    hl, vl = ln[ds.tasks[:, 0]], ln[ds.tasks[:, 1]]
    cost = np.minimum(ds.tasks[:, 2], ds.tasks[:, 3]) + np.minimum(hl - ds.tasks[:, 2], vl - ds.tasks[:, 3])
    order = np.argsort(-cost, kind="stable")
    if os.path.exists(REF_SO):
        R = Ref()
        pool = R.pool(ds.symbols, ds.offsets)
        if ds.cfg == 3:
            from paper_2304_08662_b200 import synth
            scheme = R.scheme_matrix(synth.blosum62_text(), -1, ds.x)
        else:
            scheme = R.scheme_mm(1, -1, -1, ds.x)
        return "reference", lambda: R.extend_batch(pool, scheme, ds.tasks, ds.k, ds.band,
                                                   threads=threads, order=order)
    from oracle_py import Oracle
    O = Oracle()
    s = oracle_scheme(O, ["BLOSUM62", -1, ds.x] if ds.cfg == 3 else [1, -1, -1, ds.x])
    return "oracle", lambda: O.extend_batch(ds.symbols, ds.offsets, ds.tasks, ds.k, s, ds.band,
                                            threads=threads)


def _pool(xb, ds):
    if ds.cfg == 3:
        a, c = blosum62()
        s = xb.ScoringScheme.from_matrix(xb.SubMatrix(a, c), -1, ds.x)
    else:
        s = xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x)
    return xb.DevicePool(s, ds.symbols, ds.offsets)


EXPECTED_TASKS = {1: 1_000, 2: 10_000, 3: 10_000, 4: 100_000, 5: 2_000_000}


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_config_full_size_every_row(xb, cfg):
    from paper_2304_08662_b200 import synth
    ds = synth.make(cfg, 1.0)
    assert ds.n_tasks == EXPECTED_TASKS[cfg]
    pool = _pool(xb, ds)
    out, ss = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band)
    name, run = _checker(ds)
    t0 = time.time()
    exp, ess = run()
    dt = time.time() - t0
    eq = result_rows_equal(out, exp)
    bad = np.nonzero(~eq)[0]
    assert eq.all(), f"C{cfg}: {len(bad)} of {len(eq)} sides differ from the {name}; first {bad[:5]}"
    assert (ss == ess).all(), f"C{cfg}: seed scores differ"
    # the fields result_rows_equal leaves to the status must be the defined ones
    assert (out["status"] == exp["status"]).all()
    print(f"C{cfg}: {2 * ds.n_tasks} sides, {int(out['cells'].sum())} cells identical to the "
          f"{name} ({_host_threads()} host threads, {dt:.1f}s)")
