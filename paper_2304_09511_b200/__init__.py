"""B200-native SpMV engine (COO / CSR / DIA) — drop-in for spmvkit's hot path.

Public surface mirrors the reference package (/root/reference/pkg/src/
spmvkit/__init__.py:11-93) for the hot-path modules: containers, errors,
conversions, kernels + registry + dispatch, lanes, the stencil generator and
the row-partitioned multi-GPU path.  All products run in hand-written
sm_100a kernels (libspmv_b200.so, built in-tree by `_build.build()`); there
is no CPU fallback.
"""

from .convert import (
    DiaFillPolicy,
    coo_to_csr,
    coo_to_dia,
    csr_to_coo,
    dense_to_coo,
    dia_to_coo,
    sort_coo,
    switch_format,
    to_format,
)
from .errors import (
    DeviceError,
    DimensionMismatch,
    Diverged,
    FillRatioExceeded,
    AllCandidatesFailed,
    EmptyInput,
    IndexOverflow,
    MissingBaseline,
    ParseError,
    SparseError,
    UnsupportedField,
    UnsortedInput,
    UnsupportedCombination,
)
from .formats import (
    CooMatrix,
    CsrMatrix,
    DiaMatrix,
    DynamicMatrix,
    Format,
    MatrixShape,
    as_device,
    validate,
)
from .kernels import (
    KernelRegistry,
    KernelVersion,
    default_registry,
    dispatch,
    spmv_coo_plain,
    spmv_coo_vla,
    spmv_csr_plain,
    spmv_csr_vla,
    spmv_dia_plain,
    spmv_dia_vla,
)
from .lanes import LaneConfig
from .planconfig import PlanConfig, plan_config_of, set_plan_config
from .matrixio import (
    CorpusEntry,
    gen_banded,
    gen_random_sparse,
    gen_stencil27,
    gen_stencil27_rows,
    load_entry,
    load_manifest,
    read_matrix_market,
    write_matrix_market,
)
from .cg import CgState, cg_solve
from .autotune import Measurement, PlanChoice, TuneChoice, distribution_report, measure, plan_candidates, tune, tune_plan
from .sweep import BenchRecord, compare_records, read_records, run_corpus, write_records

__version__ = "0.1.0"
