"""One assembly of a BASELINE config (for ncu captures): python tools/asm_once.py CONFIG [RERUNS]"""
import json
import sys

sys.path.insert(0, ".")
from paper_1503_07221_b200.block_system import assemble_system
from paper_1503_07221_b200.configs import get_config

cfg = get_config(int(sys.argv[1]))
A = assemble_system(cfg.mesh(), cfg.grid())
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 0):
    A._dev.rerun()
st = A._dev.stats()
print(json.dumps({k: st[k] for k in ("ms_plan", "ms_quad", "ms_finalize", "ms_pattern", "ms_total", "n_in", "units")}))
