timeout 300 python bench.py --quick --no-cpu --no-check --minplus-sweep 2048,4096 --fp64-c 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline())
for c in ('2048','4096'):
    p=d['minplus']['points'][c]; print(c, round(p['plan_frac'],4), round(p['plan_ms'],2), round(p['ms_by_kernel']['mp_prep'],2), round(p['ms_by_kernel']['mp_fold'],2))"
