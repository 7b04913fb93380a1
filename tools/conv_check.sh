mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sort_coo.py tests/test_gpu_convert.py tests/test_gpu_fuzz.py tests/test_gpu_matrixio.py -m gpu -x -q 2>&1 | tail -4
python bench.py --conversions > gpurun_out/r2d_conversions.json 2> gpurun_out/r2d_conversions.err || tail -5 gpurun_out/r2d_conversions.err
python -c "
import json
d=json.loads(open('gpurun_out/r2d_conversions.json').read().strip().splitlines()[-1])
for k,v in d.get('conversions',d).items():
    print(k, v)
"
python tools/fuzz_parity.py 60 21 1 2>&1 | tail -3
