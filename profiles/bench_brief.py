"""One-line summary of a bench.py JSON line (value, e2e, per-kernel-family ms and GB/s)."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    c = d.get("config", {})
    pk = d.get("roofline", {}).get("per_kernel", {})
    fam = " ".join(f"{k.split('(')[1].split(',')[0]}={v['ms_per_step']:.3f}ms/{v['GBps']:.0f}" for k, v in pk.items() if "(" in k)
    e2e = d.get("e2e", {}).get("value")
    print(f"{c.get('workload')} B={c.get('rows_per_gpu')} M={c.get('tile_bits')}: {d['value']:.1f} {d['unit']} "
          f"(e2e {e2e:.1f})  {d['ms_per_step']:.3f} ms/step  {fam}" if e2e else f"{c.get('workload')}: {d['value']:.1f} {fam}")
