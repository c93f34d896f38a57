"""Run bench.py over every BASELINE config and collect one JSON file + a table.

    python tools/sweep.py [--steps K] [--warmup W] [--out gpurun_out/sweep.json]
"""
import argparse
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
ORDER = ["cfg1", "cfg2", "cfg2int", "cfg3", "cfg4b1", "cfg4b4", "cfg4b16", "cfg4b64", "cfg4b256", "cfg5b1",
         "cfg5"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "sweep.json"))
    ap.add_argument("--configs", nargs="*", default=ORDER)
    a = ap.parse_args()
    rows = {}
    for c in a.configs:
        r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", c, "--steps",
                            str(a.steps), "--warmup", str(a.warmup), "--no-cpu-baseline"],
                           capture_output=True, text=True, cwd=ROOT)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        if r.returncode or not line:
            rows[c] = {"error": (r.stderr or r.stdout)[-2000:]}
            print(f"{c}: FAILED", flush=True)
            continue
        d = json.loads(line[-1])
        rows[c] = d
        rf, tc = d["roofline"], d.get("tensor_core_baseline") or {}
        print(f"{c:9s} msGeMM {d['value']:10.1f} GOP/s  step {d['ms_per_step']*1e3:8.1f} us  "
              f"LUT kernel {rf['kernel_ms']*1e3:8.1f} us  HBM {rf['frac']*100:5.1f}%  "
              f"| K4 dense {tc.get('value', float('nan')):10.1f} GOP/s "
              f"({tc.get('ms_per_step', float('nan'))*1e3:7.1f} us, HBM {tc.get('hbm_frac', float('nan'))*100:5.1f}%)",
              flush=True)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
