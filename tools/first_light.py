"""Quick first-light check on the GPU: smoke + golden c1 in each mode."""
import sys, time
sys.path.insert(0, ".")
sys.path.insert(0, "tests"); sys.path.insert(0, "tests/golden")
import numpy as np, torch
from tmas import load_case
from helpers import tolerance_report
import paper_2508_16584_b200 as tg
for name in ["residual253", "c1", "k640", "perexpert", "perexpert_t"]:
    case = load_case(name)
    layout = "nk" if case.get("b_layout") == "expert_nk" else "kn"
    cfg = tg.ProblemConfig(n=case["n"], k=case["k"], group_sizes=tuple(case["group_sizes"]))
    ops = tg.GroupedOperands(case["a_codes"], case["a_scales"], case["b_codes"], case["b_scales"], b_layout=layout)
    for mode in ["ffma2", "exact", "plain"]:
        t0 = time.time()
        run = tg.run_adaptive(cfg, ops, exact_promotion=mode == "exact", plain_staging=mode == "plain")
        torch.cuda.synchronize()
        rep = tolerance_report(run.c_bits, case["c_golden"])
        print(name, mode, rep, f"{time.time()-t0:.2f}s", flush=True)
        if rep["out_of_tol"]:
            bad = np.argwhere(run.c_bits != case["c_golden"])
            print("  first mismatches:", bad[:8].tolist())
            print("  got ", run.c_bits[bad[0][0], :8], " want", case["c_golden"][bad[0][0], :8])
