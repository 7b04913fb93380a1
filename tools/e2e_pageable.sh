# e2e through the registered callable: pinned-backed and pageable numpy x (bench's e2e block), three runs.
for i in 1 2 3; do
python bench.py --no-per-config --steps 20 --cpu-budget 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']
print('pinned', e['value'], e['ms_per_step'], 'pageable', e['pageable_x']['value'], e['pageable_x']['ms_per_step'])"
done
