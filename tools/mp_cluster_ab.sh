# mp_chain multicast A/B at C=1024 (PARPLAN_MP_CHAIN_CLUSTER 1 vs 2), with parity
for r in 1 2; do for cl in 1 2; do
  echo "== cluster $cl"
  PARPLAN_MP_CHAIN_CLUSTER=$cl timeout 300 python bench.py --quick --no-cpu --minplus-sweep 1024 --fp64-c 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); p=d['minplus']['points']['1024']
print(p['fold_frac'], p['plan_frac'], p['matches_reference'], round(p['plan_ms'],2), {k: round(v,2) for k,v in p['ms_by_kernel'].items()})"
done; done
