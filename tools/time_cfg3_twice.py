"""The cfg-2 then cfg-3 fixed-point solves in one process, twice (the bench's order), with their phases."""
import importlib.util, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
spec = importlib.util.spec_from_file_location("solve_cfg", os.path.join(ROOT, "tools", "solve_cfg.py"))
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m)
import torch
for rep in range(2):
    for c in (2, 3):
        r = m.run(c, device=0)
        free, tot = torch.cuda.mem_get_info()
        print(rep, c, round(r["wall_seconds"], 3), r["phase_seconds"], "free GB %.1f, torch reserved %.1f" % (free / 1e9, torch.cuda.memory_reserved() / 1e9), flush=True)
