"""print a one-line summary per bench JSON file"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    p = d.get("phases", {})
    c = d.get("clocks", {})
    print(f"{f}: value {d['value']:.3e} step {d['ms_per_step']:.2f} ms | upd {p.get('update_a1_a5_ms', p.get('plan_ms', 0)):.2f} "
          f"rest {p.get('restructure_ms', 0):.2f} eval {p.get('eval_ms', 0):.2f} | eval frac {d['roofline']['frac']:.3f} "
          f"hbm(restr) {d.get('roofline_hbm', {}).get('frac', 0):.2f} | idx/red kernel {p.get('redundant_kernel_vs_indexed', 0):.2f} "
          f"e2e(r+e vs idx) {p.get('redundant_e2e_vs_indexed', 0):.2f} | launches {d.get('gpu_launches')} "
          f"clk {c.get('sm_mhz')} {c.get('reasons')} n={c.get('samples')}"
          + (f" | e2e host {d['e2e']['value']:.3e}" if 'e2e' in d else "")
          + (f" | cpu {d['cpu_baseline']['value']:.3e} ({d['cpu_baseline']['cores']} cores)" if 'cpu_baseline' in d else ""))
