#!/usr/bin/env python
"""bench.py — SpMV GFLOP/s and achieved HBM GB/s vs the byte roofline.

Default workload (BASELINE.json configs[4], the one the metric's 1/2/4/8-GPU
scaling is quoted on, and the largest single-GPU config): the 27-point
stencil on a 256^3 grid, 16,777,216 rows, 449,455,096 entries, fp64, CSR
(headline) with DIA and COO reported under "per_format".  One step = one
SpMV y = A x.  Inputs (5.7 GB CSR) are far larger than L2 (126 MB), so no
flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c1|c3|c4]
  python bench.py --impl reference ...   # the reference's CPU path (oracle port)

N>1 is launched by torchrun: each rank owns a contiguous z-slab of rows
(hpcg.py:95-154 with procs (1,1,P)) and exchanges one x plane with each
neighbour over NCCL every step; time is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SpMV GFLOP/s and achieved HBM GB/s vs byte roofline per format, 1/2/4/8 B200"
UNIT = "GFLOP/s"
L2_BYTES = 126 * 1024 * 1024

CONFIGS = {
    "c5": {"workload": "27-point stencil 256^3, f64, CSR headline (+DIA, COO)", "grid": (256, 256, 256),
           "formats": ("csr", "dia", "coo")},
    "c1": {"workload": "27-point stencil 64^3, f64, CSR headline (+DIA, COO); L2 flushed between steps",
           "grid": (64, 64, 64), "formats": ("csr", "dia", "coo")},
    "c3": {"workload": "Zipf(1.8) 2M x 2M, rows 1..50000, f64, CSR headline (+COO, f32)", "formats": ("csr", "coo")},
    "c4": {"workload": "banded 2^23 rows, 11 diagonals, N(0,1), f64, DIA headline (+CSR)", "formats": ("dia", "csr")},
}


# Random 8-byte gathers per second a B200 serves with a coalesced index and
# value stream beside them (tools/gather_ceiling.cu, profiles/r1_gather_ceiling.txt).
GATHER_CEILING_GS = 248.0


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


def algo_bytes(fmt: str, nrows: int, ncols: int, nnz: int, sv: int, ndiags: int = 0) -> int:
    """Minimum-byte model: values + indices + x once + y once."""
    if fmt == "csr":
        return nnz * (sv + 4) + (nrows + 1) * 4 + ncols * sv + nrows * sv
    if fmt == "coo":
        return nnz * (sv + 8) + ncols * sv + nrows * sv
    return nrows * ndiags * sv + ndiags * 4 + ncols * sv + nrows * sv


EXCHANGE = {"c5": "NCCL halo exchange of x planes", "c1": "NCCL halo exchange of x planes",
            "c4": "NCCL halo exchange of 4096-entry x blocks", "c3": "NCCL all-gather of x"}


def config_block(cfg_name: str, fmt: str, nrows: int, nnz: int, world: int) -> dict:
    """The `config` object of a JSON line; both arms (ours, reference) emit
    exactly this for the same run, so the driver sees the same config."""
    cfg = CONFIGS[cfg_name]
    return {"workload": cfg["workload"], "config": cfg_name, "format": fmt, "nrows": int(nrows), "nnz": int(nnz),
            "l2": ("L2 flushed between steps (252 MB write, then read back so no dirty lines remain), outside the "
                   "timed events") if cfg_name == "c1" else "inputs larger than L2 (126 MB), no flush",
            "parallelism": "single GPU" if world == 1 else
            f"row-partition: {world} contiguous row blocks, {EXCHANGE[cfg_name]}, interior rows overlapped with "
            "the exchange"}


def stencil_nnz(nx: int, ny: int, nz: int) -> int:
    """prod(3 n_d - 2) (1 for n_d = 1), matrixio.py:170-210."""
    out = 1
    for d in (nx, ny, nz):
        out *= 3 * d - 2 if d > 1 else 1
    return out


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """NVML sampling of SM clock + clock-event reasons during a region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._thread = None
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None

    def _run(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                bits = fn(self._h)
                for b, name in self.REASONS.items():
                    if bits & b and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nvml is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ timing --
def time_steps(torch, fn, steps: int, warmup: int, flush=None, dist=None):
    """W untimed steps, barrier + sync, then K steps between CUDA events on
    the launching stream.  With `flush`, an L2-flush write runs between
    steps outside per-step event pairs.  Returns seconds per step (max over
    ranks when distributed)."""
    for _ in range(warmup):
        fn()
    stream = torch.cuda.current_stream()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    if flush is None:
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for _ in range(steps):
            fn()
        end.record(stream)
        torch.cuda.synchronize()
        t = start.elapsed_time(end) / 1e3 / steps
    else:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in evs:
            flush()
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        t = sum(a.elapsed_time(b) for a, b in evs) / 1e3 / steps
    if dist is not None:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    return t


def l2_flusher(torch, device):
    """flush() writes a buffer twice the L2 size, then reads it back: the
    write evicts the matrix and x, the read evicts the write's dirty lines
    (their write-back would otherwise be charged to the timed SpMV)."""
    flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=device)
    flush_sink = torch.empty(1, dtype=torch.float32, device=device)

    def flush():
        flush_buf.zero_()
        torch.sum(flush_buf, dim=0, keepdim=True, out=flush_sink)
    return flush


def roofline(bytes_per_launch: int, t_launch: float, pk: dict, traffic=None) -> dict:
    achieved = bytes_per_launch / t_launch / 1e9
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / pk["hbm_gbs"], 4), "peak_source": pk["source"], "traffic": traffic}


def traffic_for(key: str):
    """DRAM bytes per launch from the committed ncu capture, if present."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(key)
    except Exception:
        return None


# ------------------------------------------------------------ workloads --
def build_workload(torch, sp, cfg_name: str, device):
    """Device containers + x for a config.  Returns dict fmt -> container."""
    from paper_2304_09511_b200 import synthetic
    cfg = CONFIGS[cfg_name]
    mats = {}
    if cfg_name in ("c5", "c1"):
        csr = sp.gen_stencil27(*cfg["grid"])
        mats["csr"] = csr
        if "coo" in cfg["formats"] or "dia" in cfg["formats"]:
            coo = sp.csr_to_coo(csr)
            if "dia" in cfg["formats"]:
                mats["dia"] = sp.coo_to_dia(coo)
            if "coo" in cfg["formats"]:
                mats["coo"] = coo
            else:
                del coo
    elif cfg_name == "c3":
        irp, cols, vals = synthetic.zipf_csr(2_000_000, 2_000_000, synthetic.ZIPF_SEED)
        csr = sp.CsrMatrix.from_arrays(2_000_000, 2_000_000, irp, cols, vals)
        mats["csr"] = csr
        mats["coo"] = sp.csr_to_coo(csr)
        mats["csr_f32"] = sp.CsrMatrix.from_arrays(2_000_000, 2_000_000, irp, cols, vals.astype(np.float32))
    elif cfg_name == "c4":
        n = 1 << 23
        offs, vals, nnz = synthetic.banded_dia(n, synthetic.BANDED_OFFSETS, synthetic.BANDED_SEED)
        dia = sp.DiaMatrix(sp.MatrixShape(n, n, nnz), offs, vals)
        mats["dia"] = dia
        mats["csr"] = sp.to_format(dia, "csr")
    n = next(iter(mats.values())).ncols
    x = torch.from_numpy(synthetic.probe_x(n, synthetic.X_SEED)).to(device)
    # experiment scripts (tools/*.sh) pass kernel choices as SPMV_* variables;
    # they become each container's plan configuration (never read otherwise)
    from paper_2304_09511_b200.planconfig import AUTO, PlanConfig, set_plan_config
    forced = PlanConfig.from_env()
    if forced != AUTO:
        for m in mats.values():
            set_plan_config(m, forced)
    return mats, x


def spmv_fn(sp, fmt: str):
    return {"csr": sp.spmv_csr_plain, "coo": sp.spmv_coo_plain, "dia": sp.spmv_dia_plain}[fmt.split("_")[0]]


def launches_per_spmv(sp, m) -> int:
    from paper_2304_09511_b200 import kernels as K
    if m.format == sp.Format.CSR:
        return K.csr_plan(m).info()["launches"]
    if m.format == sp.Format.COO:
        return K.coo_plan(m).info()["launches"]
    return 1


def plan_of(sp, m) -> dict:
    """Kernel configuration the plan chose (tile entries, consumer groups)."""
    from paper_2304_09511_b200 import kernels as K
    if m.format == sp.Format.CSR:
        i = K.csr_plan(m).info()
        if i["kernel"] in ("warp_stream", "panel"):
            return {"kernel": i["kernel"], "warps": i["warps"]}
        return {"tile": i["tile"], "groups": i["groups"]}
    if m.format == sp.Format.COO:
        i = K.coo_plan(m).info()
        if i["kernel"] in ("warp_stream", "panel"):
            return {"kernel": i["kernel"], "warps": i["warps"]}
        if i["kernel"] == "csr_view":  # row pointers over the sorted rows: the CSR tile kernel, +0.0 seed
            return {"kernel": "csr_view"}
        return {"tile": i["tile"], "groups": i["groups"]}
    return {}


def bytes_of(m, fmt) -> int:
    sv = m.values.element_size()
    nd = m.ndiags if fmt.startswith("dia") else 0
    rows = m.nrows
    return algo_bytes(fmt.split("_")[0], rows, m.ncols, m.nnz, sv, nd)


# ------------------------------------------------------------ cpu baseline --
def cpu_baseline_csr(irp, cols, vals, x, budget_s: float = 10.0, y_check=None) -> dict:
    """C restatement of spmv_csr_plain (oracle/spmv_oracle.c), all host threads,
    repeated until the time budget is spent.  Optionally checks the GPU y."""
    from oracle import c_oracle
    nrows = irp.shape[0] - 1
    threads = c_oracle.max_threads()
    t0 = time.perf_counter()
    y = c_oracle.csr_plain(nrows, irp, cols, vals, x)
    first = time.perf_counter() - t0
    reps = max(1, min(20, int(budget_s / max(first, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(reps):
        c_oracle.csr_plain(nrows, irp, cols, vals, x)
    t = (time.perf_counter() - t0) / reps
    out = {"value": round(2.0 * vals.shape[0] / t / 1e9, 3), "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"full matrix ({vals.shape[0]} entries), {reps} SpMVs, oracle/spmv_oracle.c csr_plain "
                     f"(OpenMP rows, same summation order as kernels.py:69-82)",
           "s_per_spmv": round(t, 4)}
    if y_check is not None:
        same = y.view(np.uint64) == y_check.view(np.uint64)
        err = np.abs(y_check - y) / np.maximum(np.abs(y), 1.0)
        out["gpu_vs_oracle"] = {"bit_exact": bool(same.all()), "bit_exact_rows_frac": round(float(same.mean()), 6),
                                "max_rel_err": float(err.max()) if err.size else 0.0}
    return out


# ------------------------------------------------------------ conversions --
def conversions_measure(torch, sp, mats, pk, reps: int = 3) -> dict:
    """SURVEY.md §8(a) rows G1 and C1c-C5c at the bench config: each public
    conversion timed with CUDA events (warm-up 1, median of `reps`), with
    its minimum-byte model (containers are copied, like convert.py; two-pass
    conversions read their indices twice)."""
    from paper_2304_09511_b200 import convert as C
    from paper_2304_09511_b200 import matrixio as M
    csr = mats["csr"]
    n, nnz, sv = csr.nrows, csr.nnz, csr.values.element_size()
    coo = C.csr_to_coo(csr)
    dia = C.coo_to_dia(coo)
    nd, prow = dia.ndiags, dia.values.shape[0]
    gen_args = CONFIGS["c5"]["grid"] if n == 256 ** 3 else None
    g = torch.Generator(device=csr.values.device)
    g.manual_seed(7)
    perm = torch.randperm(nnz, device=csr.values.device, generator=g)
    shuffled = sp.CooMatrix(coo.shape, coo.row_indices[perm], coo.col_indices[perm], coo.values[perm], sorted=False)
    del perm
    # a row-stable shuffle: sort the random permutation by row (stable), so
    # rows stay in order and each row's entries are permuted
    key = coo.row_indices.to(torch.int64) * nnz + torch.randperm(nnz, device=csr.values.device, generator=g)
    order = torch.argsort(key)
    del key
    rows_ordered = sp.CooMatrix(coo.shape, coo.row_indices[order], coo.col_indices[order], coo.values[order],
                                sorted=False)
    del order
    idx = 4 * nnz
    cases = {
        # name: (callable, algorithmic bytes)
        "csr_to_coo": (lambda: C.csr_to_coo(csr), 4 * (n + 1) + nnz * (4 + sv) + nnz * (8 + sv)),
        "coo_to_csr": (lambda: C.coo_to_csr(coo), nnz * (8 + sv) + 4 * (n + 1) + nnz * (4 + sv)),
        "coo_to_dia": (lambda: C.coo_to_dia(coo), 2 * idx + nnz * (8 + sv) + prow * nd * sv),
        "dia_to_coo": (lambda: C.dia_to_coo(dia), 2 * prow * nd * sv + nnz * (8 + sv)),
        "sort_coo": (lambda: C.sort_coo(shuffled), 2 * nnz * (8 + sv)),
        # rows in order, columns shuffled inside each row, flag unset: the
        # within-row sort only (no row sort, no random gathers)
        "sort_coo_rows_ordered": (lambda: C.sort_coo(rows_ordered), 2 * nnz * (8 + sv)),
    }
    if gen_args is not None:
        cases["gen_stencil27"] = (lambda: M.gen_stencil27(*gen_args), 4 * (n + 1) + nnz * (4 + sv))
    out = {}
    stream = torch.cuda.current_stream()
    for name, (fn, b) in cases.items():
        r = fn()
        del r
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            r = fn()
            e.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(e) / 1e3)
            del r
        t = sorted(ts)[len(ts) // 2]
        out[name] = {"ms": round(t * 1e3, 3), "bytes": int(b), "gbs": round(b / t / 1e9, 1),
                     "roofline_frac": round(b / t / 1e9 / pk["hbm_gbs"], 4)}
    out["_note"] = ("event-timed public calls (incl. host syncs of the analyze steps); bytes = minimum model: "
                    "outputs written once, inputs read once per pass")
    return out


# ------------------------------------------------------------------- ours --
def run_ours(args, torch, dist, rank, world, local_rank):
    import paper_2304_09511_b200 as sp
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    pk = peaks()
    cfg = CONFIGS[args.config]
    if world > 1 or args.force_dist:
        return run_ours_multi(args, torch, dist, rank, world, local_rank, pk)
    mats, x = build_workload(torch, sp, args.config, device)
    if args.conversions:
        emit({"config": args.config, "conversions": conversions_measure(torch, sp, mats, pk)})
        return
    flush = l2_flusher(torch, device) if args.config == "c1" else None
    results = {}
    head = args.format or cfg["formats"][0]
    clocks = None
    order = [head] + [f for f in mats if f != head]
    for fmt in ([head] if args.no_extras else order):
        m = mats[fmt]
        y = torch.empty(m.nrows, dtype=m.values.dtype, device=device)
        fn_ = spmv_fn(sp, fmt)
        xx = x if m.values.dtype == torch.float64 else x.float()
        fn = lambda: fn_(m, xx, out=y)  # noqa: E731
        fn()  # plan creation (untimed, like measure()'s conversion + warm-up)
        torch.cuda.synchronize()
        if fmt == head:
            sampler = ClockSampler(local_rank)
            with sampler:
                t = time_steps(torch, fn, args.steps, args.warmup, flush)
            clocks = sampler.summary()
        else:
            t = time_steps(torch, fn, max(10, args.steps // 4), args.warmup, flush)
        b = bytes_of(m, fmt)
        results[fmt] = {"gflops": round(2.0 * m.nnz / t / 1e9, 2), "ms_per_spmv": round(t * 1e3, 4),
                        "gbs": round(b / t / 1e9, 1), "bytes_per_spmv": b, "launches": launches_per_spmv(sp, m),
                        "plan": plan_of(sp, m), "roofline_frac": round(b / t / 1e9 / pk["hbm_gbs"], 4), "nnz": m.nnz}
        if results[fmt]["plan"].get("kernel") == "csr_view":
            # COO plan without long runs: products run the CSR tile kernel on
            # the plan's row-pointer view and never read the row indices, so
            # the bytes moved are CSR's; roofline_frac above is against the COO
            # minimum-byte model of SURVEY.md 8(d) and can exceed 1
            bs = algo_bytes("csr", m.nrows, m.ncols, m.nnz, m.values.element_size(), 0)
            results[fmt].update(bytes_streamed=bs, streamed_gbs=round(bs / t / 1e9, 1),
                                streamed_frac=round(bs / t / 1e9 / pk["hbm_gbs"], 4))
            if not args.no_extras:
                # the COO tile kernel itself (segmented scan over the (row, col, value) stream)
                from paper_2304_09511_b200.planconfig import PlanConfig
                tile_cfg = PlanConfig(panels=0)
                fn_t = lambda: fn_(m, xx, out=y, plan_config=tile_cfg)  # noqa: E731
                fn_t()
                torch.cuda.synchronize()
                tt = time_steps(torch, fn_t, max(10, args.steps // 4), args.warmup, flush)
                from paper_2304_09511_b200 import kernels as K
                ti = K.coo_plan(m, config=tile_cfg).info()
                results[fmt + "_tile_kernel"] = {
                    "gflops": round(2.0 * m.nnz / tt / 1e9, 2), "ms_per_spmv": round(tt * 1e3, 4),
                    "gbs": round(b / tt / 1e9, 1), "bytes_per_spmv": b, "launches": ti["launches"],
                    "plan": {"tile": ti["tile"], "groups": ti["groups"], "config": "PlanConfig(panels=0)"},
                    "roofline_frac": round(b / tt / 1e9 / pk["hbm_gbs"], 4), "nnz": m.nnz}
        if args.config == "c3":
            # uniform random columns: every entry is one random 32-byte x
            # sector; the bound is the measured random-gather rate, not HBM
            results[fmt]["gather_roofline"] = {
                "achieved_ggathers_s": round(m.nnz / t / 1e9, 1), "ceiling_ggathers_s": GATHER_CEILING_GS,
                "frac": round(m.nnz / t / 1e9 / GATHER_CEILING_GS, 3),
                "source": "tools/gather_ceiling.cu, profiles/r1_gather_ceiling.txt (index + value stream + one "
                          "random gather per entry, best of LSU / TMA gather4 / both)",
                "note": "the ceiling of row-order kernels whose every x read is a random L2 gather; the column-panel "
                        "path (csrc/panel.cuh) reads the long rows' x from shared memory, so frac > 1 is expected"}
    vla_results = {}
    if not args.no_extras:
        # the vla kernels (kernels.py:104-210) at the reference's default lane count
        cfg_l = sp.LaneConfig()
        for fmt, m in mats.items():
            if fmt not in ("csr", "coo", "dia"):
                continue
            fn_ = {"csr": sp.spmv_csr_vla, "coo": sp.spmv_coo_vla, "dia": sp.spmv_dia_vla}[fmt]
            y = torch.empty(m.nrows, dtype=m.values.dtype, device=device)
            fn = lambda: fn_(m, x, cfg_l, out=y)  # noqa: E731
            fn()
            torch.cuda.synchronize()
            t = time_steps(torch, fn, max(10, args.steps // 4), args.warmup, flush)
            b = bytes_of(m, fmt)
            vla_results[fmt] = {"lanes": cfg_l.lanes, "gflops": round(2.0 * m.nnz / t / 1e9, 2),
                                "ms_per_spmv": round(t * 1e3, 4), "gbs": round(b / t / 1e9, 1),
                                "roofline_frac": round(b / t / 1e9 / pk["hbm_gbs"], 4)}
    m = mats[head]
    t = results[head]["ms_per_spmv"] / 1e3
    line = {
        "metric": METRIC, "value": results[head]["gflops"], "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": results[head]["ms_per_spmv"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json configs)",
        "config": config_block(args.config, head, m.nrows, m.nnz, 1),
        "roofline": roofline(results[head]["bytes_per_spmv"], t, pk, traffic_for(f"{args.config}/{head}")),
        "gpu_launches": args.steps * results[head]["launches"],
        "clocks": clocks,
        "per_format": results,
    }
    if vla_results:
        line["per_format_vla"] = vla_results
    if not args.no_extras:
        line["e2e"] = e2e_measure(args, torch, sp, m, x, head)
        if "csr" in mats and "dia" in mats:  # Zipf has no DIA form (fill ratio)
            line["conversions"] = conversions_measure(torch, sp, mats, pk)
        if args.config == "c5":
            line["cg"] = cg_measure(torch, sp, mats["csr"], pk)
        if args.config in ("c5", "c1", "c3", "c4"):
            csr = mats["csr"]
            h = csr.to_host()
            y_gpu = sp.spmv_csr_plain(csr, x).cpu().numpy()
            line["cpu_baseline"] = cpu_baseline_csr(h["row_pointers"], h["col_indices"], h["values"],
                                                    x.cpu().numpy(), args.cpu_budget, y_check=y_gpu)
            del h, y_gpu
    if not args.no_extras and args.config == "c5" and args.per_config:
        # the other large configs under the same clock (BASELINE.json configs
        # 3 and 4): device memory of the 256^3 containers is released first
        del mats, m, x
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        line["per_config"] = {c: per_config_measure(args, torch, sp, device, pk, c) for c in ("c3", "c4", "c1")}
    emit(line)


def _oracle_check(y_gpu: np.ndarray, ref: np.ndarray, exact_rows=None) -> dict:
    """GPU y against the C oracle's y: bit-exact row fraction, max rel_err
    (tests/helpers.py:71-77 semantics), and whether every row that is
    required to be bit-exact (exact_rows mask) is."""
    ui = np.uint64 if y_gpu.dtype.itemsize == 8 else np.uint32
    same = y_gpu.view(ui) == ref.astype(y_gpu.dtype).view(ui)
    err = np.abs(y_gpu.astype(np.float64) - ref.astype(np.float64)) / np.maximum(np.abs(ref.astype(np.float64)), 1.0)
    out = {"bit_exact_rows_frac": round(float(same.mean()), 6), "max_rel_err": float(err.max()) if err.size else 0.0}
    if exact_rows is not None:
        out["required_bit_exact_rows_ok"] = bool(same[exact_rows].all())
    return out


def per_config_measure(args, torch, sp, device, pk, name: str) -> dict:
    """One config of BASELINE.json besides the headline: every format's
    device-timed GFLOP/s and roofline fraction, plus its y against the C
    oracle (oracle/spmv_oracle.c) on the same inputs."""
    from oracle import c_oracle
    mats, x = build_workload(torch, sp, name, device)
    xh = x.cpu().numpy()
    steps = max(10, args.steps)
    out = {"workload": CONFIGS[name]["workload"]}
    flush = None
    if name == "c1":  # fits in L2: flushed between steps, outside the per-step event pairs
        flush = l2_flusher(torch, device)
        steps = max(10, args.steps // 4)
        out["l2"] = "L2 flushed between steps (252 MB write, then read back), outside the timed events"
    refs = {}
    csr_h = mats["csr"].to_host()
    irp = csr_h["row_pointers"]
    short = np.diff(irp.astype(np.int64)) <= 32  # rows the kernels keep in the reference order
    refs["csr"] = c_oracle.csr_plain(len(irp) - 1, irp, csr_h["col_indices"], csr_h["values"], xh)
    if "dia" in mats:
        hd = mats["dia"].to_host()
        refs["dia"] = c_oracle.dia_plain(mats["dia"].nrows, mats["dia"].ncols, hd["offsets"], hd["values"], xh)
        del hd
    for fmt, m in mats.items():
        y = torch.empty(m.nrows, dtype=m.values.dtype, device=device)
        fn_ = spmv_fn(sp, fmt)
        xx = x if m.values.dtype == torch.float64 else x.float()
        fn = lambda: fn_(m, xx, out=y)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        t = time_steps(torch, fn, steps, args.warmup, flush)
        b = bytes_of(m, fmt)
        r = {"gflops": round(2.0 * m.nnz / t / 1e9, 2), "ms_per_spmv": round(t * 1e3, 4),
             "gbs": round(b / t / 1e9, 1), "bytes_per_spmv": b, "launches": launches_per_spmv(sp, m),
             "plan": plan_of(sp, m), "roofline_frac": round(b / t / 1e9 / pk["hbm_gbs"], 4), "nnz": m.nnz,
             "steps": steps}
        if flush is not None:
            # back-to-back products: the 64^3 operator (87 MB CSR) stays in the
            # 126 MB L2, which is how a solver iteration sees it; reported
            # beside the flushed number, never as the roofline figure
            tw = time_steps(torch, fn, steps * 4, args.warmup)
            r["l2_resident"] = {"gflops": round(2.0 * m.nnz / tw / 1e9, 2), "ms_per_spmv": round(tw * 1e3, 4),
                                "gbs": round(b / tw / 1e9, 1),
                                "note": "back-to-back, no flush: matrix and x served from L2; not an HBM roofline number"}
            # the same 100 products as one CUDA graph: eager launches of a ~13 us
            # product are bound by the host's launch rate, a graph replay is not
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                for _ in range(100):
                    fn()
            graph.replay()
            torch.cuda.synchronize()
            tg = time_steps(torch, graph.replay, 10, 3) / 100
            r["l2_resident"].update({"graph_gflops": round(2.0 * m.nnz / tg / 1e9, 2),
                                     "graph_ms_per_spmv": round(tg * 1e3, 4),
                                     "graph_note": "100 products captured in one CUDA graph, replayed 10 times"})
            del graph
        if name == "c3":
            r["gather_roofline"] = {
                "achieved_ggathers_s": round(m.nnz / t / 1e9, 1), "ceiling_ggathers_s": GATHER_CEILING_GS,
                "frac": round(m.nnz / t / 1e9 / GATHER_CEILING_GS, 3),
                "source": "tools/gather_ceiling.cu, profiles/r1_gather_ceiling.txt",
                "note": "ceiling of row-order kernels (every x read a random L2 gather); the column-panel path reads "
                        "the long rows' x from shared memory, so frac > 1 is expected"}
        yg = y.cpu().numpy()
        if fmt.startswith("dia"):
            r["gpu_vs_oracle"] = _oracle_check(yg, refs["dia"], np.ones(m.nrows, dtype=bool))
        elif fmt.endswith("f32"):
            # fp32 bar: 1e-5 against the f64-evaluated product
            r["gpu_vs_oracle"] = _oracle_check(yg, refs["csr"])
            r["gpu_vs_oracle"]["bar"] = "f32 within 1e-5 of the f64-evaluated oracle"
        else:
            r["gpu_vs_oracle"] = _oracle_check(yg, refs["csr"], short)
        out[fmt] = r
        del y
    del mats, x
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    return out


def run_ours_multi(args, torch, dist, rank, world, local_rank, pk):
    """Row-partitioned path: rank r owns z-slab r of the stencil (hpcg.py:109
    with procs (1,1,P)), exchanges x halo planes over NCCL every step with
    the interior rows overlapping the exchange; time = max over ranks."""
    import paper_2304_09511_b200 as sp
    from paper_2304_09511_b200 import synthetic
    from paper_2304_09511_b200.dist import DistributedMatrix, RowPartition, _csr_rows
    from paper_2304_09511_b200.matrixio import stencil27_nnz

    device = torch.device("cuda", local_rank)
    cfg = CONFIGS[args.config]
    nd = 27
    if args.config in ("c5", "c1"):
        # z-slabs of the stencil, generated per rank on the device
        nx, ny, nz = cfg["grid"]
        n = nx * ny * nz
        nnz_total = stencil27_nnz(nx, ny, nz)
        part = RowPartition.contiguous(n, world, unit=nx * ny)
        r0, r1 = part.rows(rank)
        rows = sp.gen_stencil27_rows(nx, ny, nz, r0, r1)
    elif args.config == "c4":
        # banded 2^23: row blocks (multiples of ROW_PAD), 4096-entry halos
        n = 1 << 23
        offs, vals, nnz_total = synthetic.banded_dia(n, synthetic.BANDED_OFFSETS, synthetic.BANDED_SEED)
        nd = len(offs)
        part = RowPartition.contiguous(n, world, unit=8)
        r0, r1 = part.rows(rank)
        # only this rank's rows go to the device: the slab's DIA rows with
        # offsets shifted by r0 (column - local row) hold its global columns
        slab = sp.DiaMatrix(sp.MatrixShape(r1 - r0, n, int(np.count_nonzero(vals[r0:r1]))),
                            (offs.astype(np.int64) + r0).astype(np.int32), np.ascontiguousarray(vals[r0:r1]))
        rows = sp.to_format(slab, "csr")
        del slab
    else:
        # Zipf: every rank needs all of x (uniform columns): NCCL all-gather
        n = 2_000_000
        irp, cols, vals = synthetic.zipf_csr(n, n, synthetic.ZIPF_SEED)
        nnz_total = int(irp[-1])
        part = RowPartition.contiguous(n, world)
        r0, r1 = part.rows(rank)
        e0, e1 = int(irp[r0]), int(irp[r1])
        rows = sp.CsrMatrix.from_arrays(r1 - r0, n, (irp[r0:r1 + 1].astype(np.int64) - e0).astype(np.uint32),
                                        cols[e0:e1], vals[e0:e1])
    x_full = synthetic.probe_x(n, synthetic.X_SEED)
    x_local = torch.from_numpy(x_full[r0:r1]).to(device)
    head = args.format or cfg["formats"][0]
    fmts = [head] if args.no_extras else [head] + [f for f in cfg["formats"] if f != head]
    results, clocks, dms = {}, None, {}
    for fmt in fmts:
        dm = DistributedMatrix.build(rows, part, rank, fmt)
        dms[fmt] = dm
        dm.x_local.copy_(x_local)
        y = torch.empty(r1 - r0, dtype=torch.float64, device=device)
        fn = lambda: dm.spmv(out=y)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        if fmt == head:
            sampler = ClockSampler(local_rank)
            with sampler:
                t = time_steps(torch, fn, args.steps, args.warmup, dist=dist)
            clocks = sampler.summary()
        else:
            t = time_steps(torch, fn, max(10, args.steps // 4), args.warmup, dist=dist)
        b_total = algo_bytes(fmt, n, n, nnz_total, 8, nd)
        agg = b_total / t / 1e9
        results[fmt] = {"gflops": round(2.0 * nnz_total / t / 1e9, 2), "ms_per_spmv": round(t * 1e3, 4),
                        "gbs": round(agg, 1), "bytes_per_spmv": b_total, "launches": dm.launches_per_spmv(),
                        "roofline_frac": round(agg / (world * pk["hbm_gbs"]), 4), "nnz": nnz_total,
                        "halo_entries_per_rank": dm.plan.recv_entries}
    t = results[head]["ms_per_spmv"] / 1e3
    line = {
        "metric": METRIC, "value": results[head]["gflops"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": results[head]["ms_per_spmv"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json configs)",
        "config": config_block(args.config, head, n, nnz_total, world),
        "roofline": roofline(results[head]["bytes_per_spmv"] // world, t, pk, traffic_for(f"{args.config}/{head}")),
        "gpu_launches": args.steps * results[head]["launches"],
        "clocks": clocks,
        "per_format": results,
    }
    if not args.no_extras:
        dm = dms[head]
        fn_e2e_x = x_local.cpu().pin_memory()
        yh = torch.empty(r1 - r0, dtype=torch.float64).pin_memory()
        y = torch.empty(r1 - r0, dtype=torch.float64, device=device)

        def e2e_step():
            dm.x_local.copy_(fn_e2e_x, non_blocking=True)
            dm.spmv(out=y)
            yh.copy_(y, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        steps = max(5, min(args.steps, 30))
        te = time_steps(torch, e2e_step, steps, 3, dist=dist)
        line["e2e"] = {"value": round(2.0 * nnz_total / te / 1e9, 2), "unit": UNIT,
                       "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": n * 8, "ms_per_step": round(te * 1e3, 3),
                       "path": "DistributedMatrix.spmv per rank, pinned host x slice in, pinned host y slice out"}
        # parity of the row-partitioned product: every format's y gathered
        # over the group (gather_global) against the C oracle of the whole
        # matrix, on rank 0
        from paper_2304_09511_b200.dist import gather_global
        ref = None
        if rank == 0:
            from oracle import c_oracle
            if args.config in ("c5", "c1"):
                g_irp, g_cols, g_vals = c_oracle.stencil27_rows(*cfg["grid"], 0, n)
                ref = c_oracle.csr_plain(n, g_irp, g_cols, g_vals, x_full)
                lens = np.diff(g_irp.astype(np.int64))
                del g_irp, g_cols, g_vals
            elif args.config == "c4":
                ref = c_oracle.dia_plain(n, n, offs, vals, x_full)
                lens = np.zeros(n, dtype=np.int64)
            else:
                ref = c_oracle.csr_plain(n, irp, cols, vals, x_full)
                lens = np.diff(irp.astype(np.int64))
        parity = {}
        for fmt, dm in dms.items():
            yy = torch.empty(r1 - r0, dtype=torch.float64, device=device)
            dm.spmv(out=yy)
            g = gather_global(part, yy)
            if rank == 0:
                parity[fmt] = _oracle_check(g.cpu().numpy(), ref, lens <= 32)
        if rank == 0:
            line["gpu_vs_oracle"] = parity
    if rank == 0:
        emit(line)


def cg_measure(torch, sp, m, pk, iters: int = 20) -> dict:
    """The reference's HPCG vehicle (hpcg.py:211-258) on the device: CG with
    a fixed iteration count (tol 0) on A x = A 1, device-timed; two host
    syncs per iteration for p.Ap and r.r, as in the reference."""
    b = sp.spmv_csr_plain(m, torch.ones(m.ncols, dtype=m.values.dtype, device=m.values.device))
    sp.cg_solve(m, b, tol=0.0, max_iters=2)  # warm-up (plans, workspaces)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = sp.cg_solve(m, b, tol=0.0, max_iters=iters)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / st.iterations
    # per iteration: one SpMV + p.Ap (2 reads) + fused x/r update and r.r
    # (3 reads, 2 writes) + p = r + beta p (2 reads, 1 write) = 10 vectors
    vec_bytes = 10 * m.nrows * m.values.element_size()
    b_iter = bytes_of(m, "csr") + vec_bytes
    return {"iterations": st.iterations, "ms_per_iter": round(t * 1e3, 4),
            "spmv_gflops_equiv": round(2.0 * m.nnz / t / 1e9, 2), "gbs": round(b_iter / t / 1e9, 1),
            "roofline_frac": round(b_iter / t / 1e9 / pk["hbm_gbs"], 4),
            "relative_residual": st.relative_residual,
            "note": "cg.cg_solve (hpcg.cg_solve semantics), CSR plain; bytes = matrix + 10 vector passes"}


def e2e_measure(args, torch, sp, m, x, fmt) -> dict:
    """The reference's calling convention end to end: the GPU callable
    registered into a KernelRegistry (plugin.register_gpu_kernels, the
    kernels.py:213-244 interface) called as fn(matrix, numpy x, config) and
    returning a fresh numpy y, every step.  x is a numpy array over pinned
    host memory (the contract's "inputs from pinned host memory"), y comes
    back in pinned memory; the library pipelines upload / product /
    download (csrc/hostpipe.cuh).  Also timed: the same call with a plain
    pageable numpy x (staged by the library's pinned ring)."""
    from paper_2304_09511_b200.kernels import KernelRegistry
    from paper_2304_09511_b200.plugin import register_gpu_kernels
    reg = register_gpu_kernels(KernelRegistry())
    fn = reg.lookup(fmt.split("_")[0], "plain")
    pinned = torch.empty(m.ncols, dtype=m.values.dtype, pin_memory=True)
    pinned.copy_(x.to(m.values.dtype).cpu())
    x_np = pinned.numpy()  # numpy over pinned memory
    x_pageable = x_np.copy()
    steps = max(5, min(args.steps, 30))
    out = {}
    for name, xh in (("pinned", x_np), ("pageable", x_pageable)):
        for _ in range(3):
            y = fn(m, xh, None)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            y = fn(m, xh, None)
        wall = (time.perf_counter() - t0) / steps
        assert isinstance(y, np.ndarray) and y.shape == (m.nrows,)
        out[name] = wall
        del y
    sv = m.values.element_size()
    t = out["pinned"]
    return {"value": round(2.0 * m.nnz / t / 1e9, 2), "unit": UNIT, "h2d_bytes_per_step": m.ncols * sv,
            "d2h_bytes_per_step": m.nrows * sv, "ms_per_step": round(t * 1e3, 3), "steps": steps,
            "timing": "host wall clock around each blocking call (it returns a numpy y: the step is synchronous)",
            "path": f"register_gpu_kernels(KernelRegistry()).lookup('{fmt.split('_')[0]}', 'plain')"
                    "(A, numpy x over pinned memory, None) -> fresh numpy y (pinned)",
            "pageable_x": {"value": round(2.0 * m.nnz / out["pageable"] / 1e9, 2),
                           "ms_per_step": round(out["pageable"] * 1e3, 3),
                           "path": "same call with a pageable numpy x (library-staged)"}}


# -------------------------------------------------------------- reference --
def _reference_sample(args, c_oracle, synthetic):
    """The bounded CPU sample of the config's headline workload: returns
    (step function, entries per step, description, format).  A sample is a
    contiguous block of rows sized so that one step takes ~0.25 s."""
    cfg = CONFIGS[args.config]

    def calibrate(build, total_rows, unit):
        # time a 1/16 sample after a warm-up call (thread-pool start-up),
        # then size the step for ~0.25 s
        k = max(unit, total_rows // 16 // unit * unit)
        fn, nnz, _ = build(k)
        fn()
        t0 = time.perf_counter()
        fn()
        per_row = (time.perf_counter() - t0) / k
        k = int(max(unit, min(total_rows, 0.25 / max(per_row, 1e-12)))) // unit * unit
        return build(max(unit, k))

    if args.config in ("c5", "c1"):
        nx, ny, nz = cfg["grid"]
        n, plane = nx * ny * nz, nx * ny
        x = synthetic.probe_x(n, synthetic.X_SEED)

        def build(k):
            planes = k // plane
            r0 = (nz // 2 - planes // 2) * plane if planes < nz else 0
            r1 = r0 + planes * plane
            irp, cols, vals = c_oracle.stencil27_rows(nx, ny, nz, r0, r1)
            desc = (f"z-planes {r0 // plane}..{r1 // plane - 1} of the {nx}x{ny}x{nz} stencil "
                    f"({r1 - r0} rows, {vals.shape[0]} entries) per step; oracle/spmv_oracle.c csr_plain "
                    "(restates kernels.py:69-82)")
            return (lambda: c_oracle.csr_plain(r1 - r0, irp, cols, vals, x)), vals.shape[0], desc

        fn, nnz, desc = calibrate(build, n, plane)
        return fn, nnz, desc, "csr", (n, stencil_nnz(nx, ny, nz))
    if args.config == "c3":
        n = 2_000_000
        irp, cols, vals = synthetic.zipf_csr(n, n, synthetic.ZIPF_SEED)
        x = synthetic.probe_x(n, synthetic.X_SEED)

        def build(k):
            e = int(irp[k])
            sirp, scols, svals = irp[:k + 1], cols[:e], vals[:e]
            desc = (f"rows 0..{k - 1} of the Zipf matrix ({e} entries) per step; oracle/spmv_oracle.c csr_plain "
                    "(restates kernels.py:69-82)")
            return (lambda: c_oracle.csr_plain(k, sirp, scols, svals, x)), e, desc

        fn, nnz, desc = calibrate(build, n, 1024)
        return fn, nnz, desc, "csr", (n, int(irp[-1]))
    # c4: banded DIA, the config's headline format
    n = 1 << 23
    offs, vals, nnz_total = synthetic.banded_dia(n, synthetic.BANDED_OFFSETS, synthetic.BANDED_SEED)
    x = synthetic.probe_x(n, synthetic.X_SEED)
    o64 = offs.astype(np.int64)

    def build(k):
        cells = int(np.maximum(0, np.minimum(k, n - o64) - np.maximum(0, -o64)).sum())
        sv = np.ascontiguousarray(vals[:k])
        desc = (f"rows 0..{k - 1} of the banded matrix ({cells} in-bounds cells) per step; oracle/spmv_oracle.c "
                "dia_plain (restates kernels.py:85-101)")
        return (lambda: c_oracle.dia_plain(k, n, offs, sv, x)), cells, desc

    fn, nnz, desc = calibrate(build, n, 8)
    return fn, nnz, desc, "dia", (n, nnz_total)


def _reference_numpy(args, c_oracle, synthetic):
    """The unmodified reference's own numpy CSR kernel (spmvkit.kernels.
    spmv_csr_plain from baseline/_ref, the installed reference package) on a
    small sample of the stencil configs: the number the C port stands in for.
    Reported beside the port, never used as `value`."""
    ref_dir = ROOT / "baseline" / "_ref"
    if args.config not in ("c5", "c1"):
        return {"unavailable": "stencil configs only"}
    if not (ref_dir / "spmvkit" / "__init__.py").exists():
        return {"unavailable": "reference package not installed in baseline/_ref"}
    try:
        sys.path.insert(0, str(ref_dir))
        from spmvkit.formats import CsrMatrix
        from spmvkit.kernels import spmv_csr_plain
        nx, ny, nz = CONFIGS[args.config]["grid"]
        plane, planes = nx * ny, max(1, min(nz, 262144 // (nx * ny)))
        r0 = (nz // 2 - planes // 2) * plane
        r1 = r0 + planes * plane
        irp, cols, vals = c_oracle.stencil27_rows(nx, ny, nz, r0, r1)
        x = synthetic.probe_x(nx * ny * nz, synthetic.X_SEED)
        A = CsrMatrix.from_arrays(r1 - r0, nx * ny * nz, irp, cols, vals)
        y = spmv_csr_plain(A, x)  # warm-up, and the port's parity on the sample
        same = y.tobytes() == c_oracle.csr_plain(r1 - r0, irp, cols, vals, x).tobytes()

        def med3(fn):
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
            return sorted(ts)[1]

        t = med3(lambda: spmv_csr_plain(A, x))
        out = {"value": round(2.0 * vals.shape[0] / t / 1e9, 4), "unit": UNIT, "cores": 1, "kind": "reference",
               "s_per_step": round(t, 4), "port_bit_identical_on_sample": bool(same),
               "sample": (f"z-planes {r0 // plane}..{r1 // plane - 1} of the {nx}x{ny}x{nz} stencil "
                          f"({r1 - r0} rows, {vals.shape[0]} entries); spmvkit.kernels.spmv_csr_plain "
                          "(kernels.py:69-82) from baseline/_ref, median of 3")}
        # the other two formats of the same sample (kernels.py:56-66, :85-101), the reference's own conversions
        from spmvkit.convert import DiaFillPolicy, to_format
        from spmvkit.kernels import spmv_coo_plain, spmv_dia_plain
        coo = to_format(A, "coo")
        dia = to_format(coo, "dia", DiaFillPolicy(float("inf")))
        for name, fn in (("coo", lambda: spmv_coo_plain(coo, x)), ("dia", lambda: spmv_dia_plain(dia, x))):
            fn()
            tf = med3(fn)
            out[name] = {"value": round(2.0 * vals.shape[0] / tf / 1e9, 4), "s_per_step": round(tf, 4)}
        return out
    except Exception as exc:  # a report field only: never fails the arm
        return {"unavailable": f"{type(exc).__name__}: {exc}"}
    finally:
        if sys.path and sys.path[0] == str(ref_dir):
            sys.path.pop(0)


def run_reference(args, rank, world):
    """The reference's CPU SpMV (C restatement of kernels.py, all host
    threads) on a bounded sample of the same workload; no GPU touched."""
    if rank != 0:
        return
    from oracle import c_oracle
    from paper_2304_09511_b200 import synthetic
    cfg = CONFIGS[args.config]
    fn, nnz, sample, fmt, dims = _reference_sample(args, c_oracle, synthetic)
    for _ in range(args.warmup):
        fn()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn()
    t = (time.perf_counter() - t0) / args.steps
    v = round(2.0 * nnz / t / 1e9, 3)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json configs)",
            "config": config_block(args.config, fmt, dims[0], dims[1], world),
            "cpu_baseline": {"value": v, "unit": UNIT, "kind": "port", "cores": c_oracle.max_threads(),
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_numpy": _reference_numpy(args, c_oracle, synthetic)}
    emit(line)


_JSON_FD = None


def emit(line: dict) -> None:
    """The one JSON line, on the real stdout (see main)."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def launcher_cmd(argv: list, gpus: int, port: int) -> list:
    """`bench.py --gpus N` outside torchrun (no WORLD_SIZE): the same command
    under torch.distributed.run, one rank per GPU, rendezvous on 127.0.0.1."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), *argv]


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    global _JSON_FD
    pre = argparse.ArgumentParser(add_help=False)
    pre.add_argument("--gpus", type=int, default=1)
    pre.add_argument("--print-launcher", action="store_true")
    known, _ = pre.parse_known_args()
    if known.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun; rank 0
        # prints the JSON line (n_gpus = N)
        argv = [a for a in sys.argv[1:] if a != "--print-launcher"]
        cmd = launcher_cmd(argv, known.gpus, _free_port())
        if known.print_launcher:
            print(json.dumps({"launcher": cmd}))
            return
        sys.stdout.flush()
        os.execv(cmd[0], cmd)
    # Only the JSON line goes to stdout: everything else that writes to fd 1
    # (NCCL's version banner, library chatter) is sent to stderr.
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--print-launcher", action="store_true",
                    help="with --gpus N > 1 outside torchrun: print the torchrun command instead of running it")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="c5")
    ap.add_argument("--format", default=None, help="headline format (default: the config's first)")
    ap.add_argument("--no-extras", action="store_true", help="headline format only (profiling runs)")
    ap.add_argument("--conversions", action="store_true", help="time the format conversions only")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-per-config", dest="per_config", action="store_false",
                    help="c5 only: skip the c3 / c4 / c1 lines under per_config")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the row-partitioned path even at world size 1 (exercises it on one GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    dist = None
    if world > 1 or args.force_dist:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, torch, dist, rank, world, local_rank)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
