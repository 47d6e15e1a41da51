"""Run bench.py on every BASELINE.json config (1 GPU) and print the
BASELINE.md reporting-template table (one JSON line per config, then a
markdown table).

    python tools/bench_configs.py [--gpus 1] [--steps 3] [--warmup 2]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--configs", default="1,2,3,5,4")
    args = ap.parse_args()
    rows = []
    for c in [int(x) for x in args.configs.split(",")]:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(c), "--steps",
                            str(args.steps), "--warmup", str(args.warmup), "--no-cpu-baseline"],
                           capture_output=True, text=True, cwd=ROOT)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode != 0 or not line:
            print(json.dumps({"config": c, "error": r.stderr[-2000:]}), flush=True)
            continue
        d = json.loads(line[-1])
        d["config_index"] = c
        print(json.dumps(d), flush=True)
        rows.append(d)
    print("\n| cfg | G | S5 pairs | S5 ms | S5 pairs/s | S5 K2 % bound | S2a+S2d pairs/s | partition ms | "
          "S1 % HBM | step ms | e2e pairs/s |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for d in rows:
        print(f"| {d['config_index']} | {d['n_gpus']} | {d['pairs_per_step']['S5']:,} | {d['s5_ms']:.2f} | "
              f"{d['s5_pairs_per_s']:.3g} | {100 * d['roofline']['frac']:.1f} | {d['s2_pairs_per_s_rank0']:.3g} | "
              f"{d['partition_ms']:.2f} | {100 * d['s1_hbm_rank0']['frac_of_hbm']:.1f} | {d['ms_per_step']:.2f} | "
              f"{d['e2e']['value']:.3g} |")


if __name__ == "__main__":
    main()
