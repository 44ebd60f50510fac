"""Convergence study on the GPU (SPEC.md run_convergence_study): python tools/convergence.py [out.jsonl]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09497_b200 as smg
from paper_2410_09497_b200 import harness

out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout
for k, levels in ((1, [1, 2, 3, 4, 5]), (2, [1, 2, 3, 4, 5]), (3, [1, 2, 3, 4])):
    for vp in (smg.F64, smg.F32):
        for r in harness.convergence_study([k], levels, vcycle_precision=vp):
            out.write(json.dumps(r) + "\n")
            out.flush()
