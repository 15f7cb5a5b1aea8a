for ws in 1 0; do echo ws=$ws; MI_RX_WS=$ws timeout 900 python tools/time_cfg3_twice.py 2>&1 | grep -v Warning | tail -4; done
