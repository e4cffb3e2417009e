# Chain-item row cap A/B (PARPLAN_CHAIN_ROWS; the builder's makespan model picks up to it)
for r in 1 2; do for v in 4 6 8; do echo "== rows $v"; PARPLAN_CHAIN_ROWS=$v python tools/split_ab.py 2>&1; PARPLAN_CHAIN_ROWS=$v python tools/phase_list.py inception_chain@16 vgg16@16 "inception_chain(13)@16" alexnet@4 2>&1; done; done
