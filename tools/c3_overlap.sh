# C3: short-row kernel on a side stream beside the panel kernel (SPMV_PANEL_OVERLAP=1, default) vs in sequence (=0).
mkdir -p gpurun_out
for ov in 0 1 0 1; do
  SPMV_PANEL_OVERLAP=$ov python bench.py --config c3 --no-extras --steps 200 --warmup 5 > gpurun_out/c3_ov$ov.json 2> gpurun_out/c3_ov$ov.err || { tail -5 gpurun_out/c3_ov$ov.err; exit 1; }
  python - <<PY
import json
d = json.load(open("gpurun_out/c3_ov$ov.json"))
print("overlap=$ov", {k: (v["gflops"], v["ms_per_spmv"], v["roofline_frac"]) for k, v in d["per_format"].items()})
PY
done
timeout 900 python -m pytest tests/test_gpu_panel.py tests/test_gpu_planconfig.py -m gpu -x -q 2>&1 | tail -3
