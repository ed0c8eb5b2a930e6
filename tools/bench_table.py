"""Markdown table of bench.py JSON lines (profiles/ evidence).

    python tools/bench_table.py gpurun_out/bench_configs.jsonl [default.json] > profiles/rNN_bench_configs.md
"""
import json
import sys


def rows(path):
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            yield json.loads(line)


def main():
    out = ["| config | scaling | dtype | ms / step | eff. GFLOP/s | e2e GFLOP/s | K2 kernel frac | K3 fused | step shares | clocks |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for p in sys.argv[1:]:
        for d in rows(p):
            cfg = d["config"]["workload"].split(":")[0]
            sc = "none"
            if "scaling" in d["config"]["workload"]:
                sc = d["config"]["workload"].split("scaling ")[1].split(" ")[0]
            rf = d["roofline"]
            shares = ", ".join(f"{k} {v:.3f}" for k, v in rf["step_share"].items())
            clk = d.get("clocks") or {}
            e2e = d.get("e2e") or {}
            out.append(f"| {cfg} | {sc} | {d['dtype']} | {d['ms_per_step']:.3f} | {d['value']:.0f} | "
                       f"{e2e.get('value', float('nan')):.0f} | {rf['frac']:.3f} | "
                       f"{d['config'].get('k3_fused_in_leaf_epilogue')} | {shares} | "
                       f"{clk.get('sm_mhz')} MHz {' '.join(clk.get('reasons', []))} |")
    print("\n".join(out))


if __name__ == "__main__":
    main()
