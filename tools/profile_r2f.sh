# Round-2 full captures of the final kernels beyond the c5 headline: c3 panel path, c4, conversions.
# The reports are summarised on the box (profiles/ncu_summary.py); only the JSON comes back.
mkdir -p gpurun_out/r2f_rep
cap() {  # name, kernel regex, launches to skip, bench args...
  n=$1; k=$2; sk=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s $sk -c 1 -f -o gpurun_out/r2f_rep/$n python bench.py "$@" > gpurun_out/r2f_rep/ncu_$n.log 2>&1
  tail -1 gpurun_out/r2f_rep/ncu_$n.log
}
cap c3_short_ell short_ell_kernel 2 --config c3 --no-extras --steps 3 --warmup 3 --cpu-budget 1
cap c3_panel "csr_panel_kernel" 2 --config c3 --no-extras --steps 3 --warmup 3 --cpu-budget 1
cap c3_finish csr_panel_finish_kernel 2 --config c3 --no-extras --steps 3 --warmup 3 --cpu-budget 1
cap c4_dia dia_bulk_kernel 2 --config c4 --no-extras --steps 3 --warmup 3 --cpu-budget 1
cap c4_csr csr_tile_kernel 2 --config c4 --format csr --no-extras --steps 3 --warmup 3 --cpu-budget 1
cap conv_coo_to_csr coo_to_csr_vec_kernel 2 --conversions
cap conv_csr_to_coo csr_expand_vec_kernel 2 --conversions
cap conv_dia_count dia_tiles_kernel 2 --conversions
cap conv_dia_emit dia_tiles_kernel 3 --conversions
cap conv_group_sort group_sort_kernel 2 --conversions
cap conv_sort_rows sort_rows_kernel 2 --conversions
cap conv_diag_scatter diag_scatter_kernel 2 --conversions
cap conv_diag_mark diag_mark_kernel 2 --conversions
python profiles/ncu_summary.py gpurun_out/r2f_rep/*.ncu-rep > gpurun_out/r2f_ncu_summary.json
rm -rf gpurun_out/r2f_rep gpurun_out/r2f_*.ncu-rep gpurun_out/r2d_c5_*.ncu-rep gpurun_out/c1_*.ncu-rep gpurun_out/r2b_group_sort.ncu-rep
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2f_ncu_summary.json"))
for k, v in d.items():
    print(k.split("/")[-1], v.get("time_ms"), v.get("dram_pct_peak"), v.get("dram_bytes"), v.get("issue_active_pct"), v.get("top_stalls", [])[:2])
PY
