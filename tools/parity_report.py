"""Write the parity pins (tests/pins.py) as JSON: python tools/parity_report.py OUT.json [case ...]

Runs on the GPU box; the numbers are the same ones tests/test_gpu_parity_pins.py asserts."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_23445_b200 as dfs  # noqa: E402
from tests.pins import CASES, run_case  # noqa: E402

if __name__ == "__main__":
    out = sys.argv[1]
    cases = sys.argv[2:] or list(CASES)
    rows = []
    for c in cases:
        t = time.time()
        r = run_case(c, torch, dfs)
        r["seconds"] = round(time.time() - t, 1)
        rows.append(r)
        worst = {k: (min if k in ("bit_agree", "set_overlap", "rows_equal") else max)(h[k] for h in r["heads"])
                 for k in ("score_err", "bit_agree", "set_overlap", "rows_equal", "out_err", "out_err_own")}
        print(c, json.dumps(worst), flush=True)
    with open(out, "w") as f:
        json.dump({"gpu": torch.cuda.get_device_name(0), "cases": rows}, f, indent=1)
