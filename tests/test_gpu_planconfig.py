"""Per-plan kernel configuration, the plan tuner, and concurrent use of one
plan (kernels are pure; concurrent calls on disjoint outputs
are safe).

* Every PlanConfig candidate the tuner tries computes the same y under the
  exactness contract (rows <= exact_len bit-exact with the C oracle, all
  rows within 1e-12), and the tuner attaches its winner to the container.
* Two plans of one matrix with different configurations coexist in one
  process (no process-global knobs).
* One matrix, several threads and streams at once, disjoint outputs: every
  output equals the single-stream product bit for bit (the warp-stream range
  counter, the span partials and the host-pipeline staging are per stream /
  serialised, csrc/common.cuh StreamSlots).
"""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


def _random(sp, seed, n=40_000, ncols=60_000, long_frac=0.02):
    rng = np.random.default_rng(seed)
    lens = np.where(rng.random(n) < long_frac, rng.integers(33, 3000, n), rng.integers(0, 33, n))
    irp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=irp[1:])
    cols = np.concatenate([np.sort(rng.choice(ncols, size=int(k), replace=False)) for k in lens]).astype(np.uint32)
    vals = rng.standard_normal(cols.shape[0])
    x = rng.uniform(-1, 1, ncols)
    return sp.CsrMatrix.from_arrays(n, ncols, irp, cols, vals), irp.astype(np.uint32), cols, vals, x, lens


def _check(y, ref, lens, exact_len):
    from _util import bit_equal, first_diff, rel_err
    short = lens <= exact_len
    assert bit_equal(y[short], ref[short]), first_diff(y[short], ref[short])
    assert rel_err(y, ref) <= 1e-12


@pytest.mark.parametrize("fmt", ["csr", "coo"])
def test_every_candidate_matches_oracle(sp, fmt):
    from oracle import c_oracle
    from paper_2304_09511_b200.autotune import plan_candidates
    A, irp, cols, vals, x, lens = _random(sp, 3)
    ref = c_oracle.csr_plain(A.nrows, irp, cols, vals, x)
    m = A if fmt == "csr" else sp.csr_to_coo(A)
    run = sp.spmv_csr_plain if fmt == "csr" else sp.spmv_coo_plain
    cands = plan_candidates(m)
    assert len(cands) >= 3 and cands[0] == sp.PlanConfig()
    kernels = set()
    for cfg in cands:
        y = run(m, x, plan_config=cfg)
        _check(y, ref, lens, 32)
        from paper_2304_09511_b200 import kernels as K
        p = K.csr_plan(m, config=cfg) if fmt == "csr" else K.coo_plan(m, config=cfg)
        kernels.add(p.info()["kernel"])
    # every whole-matrix kernel is among the candidates (the panel path is CSR only)
    assert kernels == ({"tile", "warp_stream", "panel"} if fmt == "csr" else {"tile", "warp_stream"})


def test_short_row_candidates_and_exact_len(sp):
    from oracle import c_oracle
    from paper_2304_09511_b200.autotune import plan_candidates
    from paper_2304_09511_b200 import kernels as K
    A, irp, cols, vals, x, lens = _random(sp, 4, long_frac=0.0)
    ref = c_oracle.csr_plain(A.nrows, irp, cols, vals, x)
    shapes = set()
    for cfg in plan_candidates(A):
        y = sp.spmv_csr_plain(A, x, plan_config=cfg)
        _check(y, ref, lens, 32)
        r = K.csr_plan(A, config=cfg).config()
        shapes.add((r.tile, r.groups))
    assert len(shapes) >= 4
    # exact_len 8 (warp-stream kernel): rows of <= 8 entries are never split
    # between warp ranges; with many ranges per warp, longer rows are; all
    # within 1e-12, short ones bit-exact.  The tile kernels keep 32.
    cfg = sp.PlanConfig(exact_len=8, warp_stream=1, ranges_per_warp=64)
    y = sp.spmv_csr_plain(A, x, plan_config=cfg)
    assert K.csr_plan(A, config=cfg).config().exact_len == 8
    _check(y, ref, lens, 8)
    cfg = sp.PlanConfig(exact_len=8, warp_stream=0)
    _check(sp.spmv_csr_plain(A, x, plan_config=cfg), ref, lens, 32)


@pytest.mark.parametrize("fmt", ["csr", "coo", "dia"])
def test_tune_plan_attaches_winner(sp, fmt):
    A = sp.gen_stencil27(24, 24, 24)
    m = {"csr": A, "coo": sp.csr_to_coo(A), "dia": sp.coo_to_dia(sp.csr_to_coo(A))}[fmt]
    x = np.random.default_rng(1).uniform(-1, 1, A.ncols)
    y0 = sp.dispatch(m, x)
    choice = sp.tune_plan(m, iterations=3, reps=2)
    assert len(choice.timings) == len(sp.plan_candidates(m)) and choice.median_seconds > 0
    assert sp.plan_config_of(m) == choice.config
    assert sp.dispatch(m, x).tobytes() == y0.tobytes()  # stencil rows: every configuration bit-exact
    # an injected clock (the reference's hook) decides the winner: the
    # third candidate is the only fast one
    ticks = iter([0.0, 5.0, 0.0, 5.0, 0.0, 5.0, 0.0, 5.0, 0.0, 1.0, 0.0, 1.0] + [0.0, 9.0] * 40)
    c2 = sp.tune_plan(m, iterations=1, reps=2, timer=lambda: next(ticks), attach=False)
    assert c2.config == sp.plan_candidates(m)[2]
    assert sp.plan_config_of(m) == choice.config  # attach=False left it alone


def test_dia_configs(sp):
    from oracle import c_oracle
    A = sp.gen_stencil27(20, 18, 16)
    d = sp.coo_to_dia(sp.csr_to_coo(A))
    h = d.to_host()
    x = np.random.default_rng(2).uniform(-1, 1, A.ncols)
    ref = c_oracle.dia_plain(d.nrows, d.ncols, h["offsets"], h["values"], x)
    for k in range(-1, 5):
        for rows in (0, 64):
            y = sp.spmv_dia_plain(d, x, plan_config=sp.PlanConfig(dia_kernel=k, dia_rows=rows))
            assert y.tobytes() == ref.tobytes(), (k, rows)


def test_two_configs_coexist(sp):
    """No process-global switch: a tile plan and a warp-stream plan of one
    matrix, used alternately, each keep their kernel."""
    from paper_2304_09511_b200 import kernels as K
    A, irp, cols, vals, x, lens = _random(sp, 5)
    a, b = sp.PlanConfig(warp_stream=0), sp.PlanConfig(warp_stream=1, ranges_per_warp=2)
    assert K.csr_plan(A, config=a).info()["kernel"] == "tile"
    assert K.csr_plan(A, config=b).info()["kernel"] == "warp_stream"
    ya, yb = sp.spmv_csr_plain(A, x, plan_config=a), sp.spmv_csr_plain(A, x, plan_config=b)
    for _ in range(3):
        assert sp.spmv_csr_plain(A, x, plan_config=a).tobytes() == ya.tobytes()
        assert sp.spmv_csr_plain(A, x, plan_config=b).tobytes() == yb.tobytes()


@pytest.mark.parametrize("fmt,cfg", [("csr", dict(warp_stream=1)), ("csr", dict(warp_stream=0)),
                                     ("coo", dict(warp_stream=1)), ("coo", dict(warp_stream=0))])
def test_one_plan_many_streams_and_threads(sp, fmt, cfg):
    """8 threads, each on its own CUDA stream, 6 products each of ONE
    matrix (one plan) into disjoint outputs, all in flight together."""
    import torch
    A, irp, cols, vals, x, lens = _random(sp, 6)
    m = A if fmt == "csr" else sp.csr_to_coo(A)
    sp.set_plan_config(m, sp.PlanConfig(**cfg))
    run = sp.spmv_csr_plain if fmt == "csr" else sp.spmv_coo_plain
    xd = torch.from_numpy(x).cuda()
    want = run(m, xd).cpu().numpy()
    nthreads, reps = 8, 6
    outs = [[torch.full((m.nrows,), float("nan"), dtype=torch.float64, device="cuda") for _ in range(reps)]
            for _ in range(nthreads)]
    barrier = threading.Barrier(nthreads)
    errors = []
    torch.cuda.synchronize()  # the NaN fills and x are ready before other streams write

    def worker(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                barrier.wait()
                for r in range(reps):
                    run(m, xd, out=outs[t][r])
            s.synchronize()
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ths = [threading.Thread(target=worker, args=(t,)) for t in range(nthreads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errors, errors
    torch.cuda.synchronize()
    for t in range(nthreads):
        for r in range(reps):
            assert outs[t][r].cpu().numpy().tobytes() == want.tobytes(), (t, r)


def test_host_pipeline_from_threads(sp):
    """spmv_csr_host (pinned host x -> pinned host y) from 4 threads at
    once on one plan: the staging is the plan's, so calls are serialised on
    the device; every result is exact."""
    import torch
    A = sp.gen_stencil27(40, 40, 40)
    xs = [torch.from_numpy(np.random.default_rng(s).uniform(-1, 1, A.ncols)).pin_memory() for s in range(4)]
    wants = [sp.spmv_csr_plain(A, x.cuda()).cpu() for x in xs]
    outs = [torch.empty(A.nrows, dtype=torch.float64).pin_memory() for _ in range(4)]
    torch.cuda.synchronize()
    errors = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    sp.spmv_csr_plain(A, xs[i], out=outs[i])
                    assert torch.equal(outs[i], wants[i])
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ths = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errors, errors


def test_vla_two_streams(sp):
    """The two-phase vla path's product buffer is per stream."""
    import torch
    from oracle import c_oracle
    A, irp, cols, vals, x, lens = _random(sp, 7, long_frac=0.05)
    want = c_oracle.csr_vla(A.nrows, irp, cols, vals, x, 4)
    xd = torch.from_numpy(x).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ys = []
    torch.cuda.synchronize()
    for s in (s1, s2, s1, s2):
        with torch.cuda.stream(s):
            ys.append(sp.spmv_csr_vla(A, xd, sp.LaneConfig(4)))
    torch.cuda.synchronize()
    for y in ys:
        assert y.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("shuffle", [False, True])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_coo_row_pointer_view(sp, shuffle, dtype):
    """COO plans without long runs run whole-matrix products on a CSR view of
    their row-sorted triples (row pointers built by the plan; the CSR tile
    kernel with a +0.0 seed): np.add.at order, bit for bit, also for an
    unsorted input (stable row sort: storage order kept) and a lone -0.0
    product (+0.0, not cumsum's -0.0).  panels=0 or a configured COO tile
    keeps the COO tile kernel; both give the same bits."""
    from _util import bit_equal, first_diff
    from oracle import c_oracle
    from paper_2304_09511_b200 import kernels as K
    rng = np.random.default_rng(31)
    n, ncols = 50_000, 70_000
    lens = rng.integers(0, 33, n)
    rows = np.repeat(np.arange(n), lens).astype(np.uint32)
    cols = np.concatenate([np.sort(rng.choice(ncols, size=int(k), replace=False)) for k in lens]).astype(np.uint32)
    vals = rng.uniform(-1, 1, rows.shape[0]).astype(dtype)
    one = np.flatnonzero(lens == 1)[0]
    vals[np.flatnonzero(rows == one)[0]] = -0.0
    x = np.abs(rng.uniform(0.1, 1, ncols)).astype(dtype)
    if shuffle:
        order = rng.permutation(rows.shape[0])
        rows, cols, vals = rows[order], cols[order], vals[order]
    A = sp.CooMatrix.from_arrays(n, ncols, rows, cols, vals, sorted=not shuffle)
    ref = c_oracle.coo_plain(n, rows, cols, vals, x, row_sorted=not shuffle)
    assert K.coo_plan(A).info()["kernel"] == "csr_view"
    y = sp.spmv_coo_plain(A, x)
    assert bit_equal(y, ref), first_diff(y, ref)
    assert y[one] == 0 and not np.signbit(y[one])
    for cfg in (sp.PlanConfig(panels=0), sp.PlanConfig(tile=1536, groups=7)):
        assert K.coo_plan(A, config=cfg).info()["kernel"] == "tile"
        assert sp.spmv_coo_plain(A, x, plan_config=cfg).tobytes() == y.tobytes()
    if not shuffle:  # vla keeps its own kernels (and refuses unsorted input like the reference)
        from oracle import spmv_oracle as O
        assert sp.spmv_coo_vla(A, x, sp.LaneConfig(8)).tobytes() == O.coo_vla(n, rows, cols, vals, x, 8).tobytes()
