# C=1024 min-plus leg of bench.py (fold / plan fractions, parity, per-kernel ms)
timeout 300 python bench.py --quick --no-cpu --minplus-sweep 1024 --fp64-c 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); p=d['minplus']['points']['1024']
print(p['fold_frac'], p['plan_frac'], p['matches_reference'], round(p['plan_ms'],2), {k: round(v,2) for k,v in p['ms_by_kernel'].items()})"
