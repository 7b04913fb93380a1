"""Every whole-matrix CSR/COO kernel on every parity case, in-process.

Plans pick the warp-stream kernel (csrc/wstream.cuh) for matrices with rows
or runs over 32 entries and the tile kernel otherwise.  A plan's kernel
choice is its `PlanConfig`, so the corpus, stress, tail-tile and
row-partition parity suites re-run here with the choice forced each way
(`using_plan_config`: a scoped per-thread default; the plan cache is keyed
by configuration, so the forced plans live beside the automatic ones).  The
warp-stream runs use 64 ranges per warp, so long rows split across many
ranges and the fix-up carries most of them, and 1 range per warp.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


def _suites(sp, dist=True):
    import test_dist as D
    import test_gpu_kernels as K
    import test_gpu_stress as S
    from _util import corpus_names
    for name in corpus_names():
        K.test_corpus_all_kernels(sp, name)
    K.test_canonical_kats_all_formats(sp)
    for name in ("pl64", "pl32", "plempty", "edges"):
        K.test_long_rows(sp, name)
    for case in S.CASES:
        for dt in (np.float64, np.float32):
            S.test_random_structures_csr_coo(sp, case, dt)
    for mod in (1, 2, 3):
        S.test_tail_tiles_and_unaligned_pointers(sp, mod)
    S.test_unsorted_coo_duplicates_at_scale(sp)
    if not dist:
        return
    for fmt in ("csr", "coo"):
        for world in (1, 3):
            D.test_emulated_ranks_bit_identical(None, fmt, world)
    D.test_emulated_ranks_random_matrix_allgather(None)


@pytest.mark.parametrize("forced", [dict(warp_stream=1, ranges_per_warp=64), dict(warp_stream=1, ranges_per_warp=1),
                                    dict(warp_stream=0), dict(warp_stream=0, tile=1024, groups=1)],
                         ids=["ws_r64", "ws_r1", "tiles", "tiles_1024x1"])
def test_forced_kernel_choice(sp, forced):
    from paper_2304_09511_b200.planconfig import PlanConfig, using_plan_config
    cfg = PlanConfig(**forced)
    with using_plan_config(cfg):
        _suites(sp)
