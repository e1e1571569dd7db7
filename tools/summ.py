"""Summarise bench JSON lines: python tools/summ.py files..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
        continue
    s = d.get("stages_ms", {})
    sc = d.get("side_chain_ms")
    print(f"{f.split('/')[-1]:32s} {d['value']/1e6:7.2f}M {d['ms_per_step']:.3f}ms frac {d['roofline']['frac']:.3f} "
          f"rt {s.get('router', 0):.3f} sh {s.get('shared_expert', 0):.3f} g1 {s.get('gemm1_swiglu', 0):.3f} "
          f"g2 {s.get('gemm2', 0):.3f} side {sc} mhz {d['clocks']['sm_mhz']}")
