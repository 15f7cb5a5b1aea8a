for ws in 1 0; do
MI_RX_WS=$ws timeout 900 python tools/solve_cfg.py --cfg 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ws=$ws', d['wall_seconds'], d['phase_seconds'])"
done
