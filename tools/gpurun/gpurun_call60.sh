for w in 2 4 8; do timeout 600 python tools/rank_cost.py --world $w --rank 1 2>&1 | tail -1 | cut -c1-700; done
