"""First-contact GPU diagnostics: each case in its own process under a timeout."""
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CASES = [
    ("gemm", {"m": 128, "n": 64, "k": 16}),
    ("gemm", {"m": 128, "n": 64, "k": 16, "prec": "tf32"}),
    ("gemm", {"m": 300, "n": 200, "k": 70}),
    ("conv", {"method": "kn2row-gpu", "N": 1, "C": 16, "H": 8, "W": 16, "M": 16, "k": 1}),
    ("conv", {"method": "kn2row-gpu", "N": 1, "C": 16, "H": 8, "W": 16, "M": 16, "k": 3}),
    ("conv", {"method": "kn2row-gpu", "N": 2, "C": 3, "H": 13, "W": 13, "M": 40, "k": 3}),
    ("conv", {"method": "kn2row-gpu", "N": 1, "C": 64, "H": 56, "W": 56, "M": 64, "k": 3}),
    ("conv", {"method": "kn2row-gpu", "N": 3, "C": 48, "H": 7, "W": 7, "M": 128, "k": 5}),
    ("conv", {"method": "kn2row-acc-gpu", "N": 2, "C": 16, "H": 13, "W": 13, "M": 32, "k": 3}),
    ("conv", {"method": "kn2row-explicit-gpu", "N": 2, "C": 16, "H": 13, "W": 13, "M": 32, "k": 3}),
    ("conv", {"method": "kn2col-gpu", "N": 2, "C": 16, "H": 13, "W": 13, "M": 32, "k": 3}),
    ("conv", {"method": "im2col-gpu", "N": 2, "C": 16, "H": 13, "W": 13, "M": 32, "k": 3}),
    ("conv", {"method": "kn2row-gpu", "N": 2, "C": 32, "H": 13, "W": 13, "M": 384, "k": 3, "prec": "tf32"}),
]
out = Path(sys.argv[1]) if len(sys.argv) > 1 else None
lines = []
for kind, args in CASES:
    try:
        p = subprocess.run([sys.executable, str(HERE / "diag_case.py"), kind, json.dumps(args)],
                           capture_output=True, text=True, timeout=120)
        res = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
        line = res[0][7:] if res else json.dumps({"kind": kind, "args": args, "rc": p.returncode,
                                                  "err": (p.stderr or p.stdout)[-800:]})
    except subprocess.TimeoutExpired:
        line = json.dumps({"kind": kind, "args": args, "timeout": True})
    print(line, flush=True)
    lines.append(line)
if out:
    out.write_text("\n".join(lines) + "\n")
