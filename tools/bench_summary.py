"""One line per bench JSON log: GB/s, ms/step, roofline and step fractions, clocks, phase times."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        ph = d.get("phases_ms", {})
        print(f"{path.split('/')[-1]:28s} {d['value']:8.1f} GB/s {d['ms_per_step']:7.3f} ms "
              f"frac={d['roofline']['frac']:.3f} step={d['roofline'].get('step_hbm_frac', 0):.3f} "
              f"clk={d['clocks']['sm_mhz']} {d['clocks']['reasons']} pass1={ph.get('pass1', 0):.2f} "
              f"rec={ph.get('reconstruct', 0):.2f} med={ph.get('step_ms', {}).get('median', 0):.2f} "
              f"max={ph.get('step_ms', {}).get('max', 0):.1f}")
