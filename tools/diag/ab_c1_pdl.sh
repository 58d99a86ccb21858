for i in 1 2; do
for v in "SYNK_F32X3_PDL=0" "SYNK_F32X3_PDL=1"; do
env $v timeout 300 python bench.py --no-c3 --no-c4 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=j['sync_sgd']; r=s['runs'][0]
print('$v', 'C1 ms', round(s['ms_per_step'],5), 'C1exact', round(j.get('sync_sgd_c1_exact',{}).get('ms_per_step',0) or 0,5), 'C5', round(j['sync_sgd_wide_bf16']['ms_per_step'],5), 'e2e', round(j['e2e']['value']))"
done; done
