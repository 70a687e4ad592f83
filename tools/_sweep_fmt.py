"""Compact one-line-per-point view of tools/sweep_c4.py JSON lines (stdin).

usage: python tools/sweep_c4.py ... | python tools/_sweep_fmt.py
"""
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r["mode"], r["layer"], r["zero_frac"], round(r["ms"],3), round(r["tflops"],2), r.get("normwise_err_vs_exact",""))
