"""Counter-derived FP64 FLOPs of a matvec kernel launch from an ncu raw-page CSV export
(`ncu -i X.ncu-rep --page raw --csv`), in the convention of ncu's FP64 roofline:
FLOPs = 2 * DFMA + DMUL + DADD thread instructions (sm__sass_thread_inst_executed_op_*_pred_on),
peak = 2 * the DFMA peak (sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained).
Writes / updates profiles/<round>/ncu_flops.json, which bench.py reads for roofline
`executed_fp64_flops_per_unit` and `ncu_fp64_flop_frac`.

Usage: python tools/ncu_flops.py RAW.csv KEY CONFIG [OUT.json]
  KEY: "1x" symmetric kernel with exact sums, "1" fixed-order partials, "0" row kernel.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def read_raw(path):
    rows = list(csv.reader(open(path)))
    i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[i0], rows[i0 + 2:]
    return [dict(zip(hdr, r)) for r in data if len(r) == len(hdr)]


def num(d, k):
    return float(str(d[k]).replace(",", ""))


def summarise(rec, n_ordered_pairs):
    cyc = num(rec, "sm__cycles_elapsed.avg")
    ops = {op: num(rec, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed") * cyc
           for op in ("dfma", "dmul", "dadd")}
    flops = 2 * ops["dfma"] + ops["dmul"] + ops["dadd"]
    peak_per_cycle = 2 * num(rec, "sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained")
    return {"kernel": rec.get("Kernel Name"), "duration_ms": num(rec, "gpu__time_duration.sum"),
            "sm_clock_ghz": num(rec, "sm__cycles_elapsed.avg.per_second"),
            "fp64_flops_per_launch": flops, "ordered_pairs_per_launch": n_ordered_pairs,
            "fp64_flops_per_ordered_pair": flops / n_ordered_pairs,
            "fp64_instr_per_ordered_pair": {k: v / n_ordered_pairs for k, v in ops.items()},
            "ncu_fp64_flop_frac": flops / cyc / peak_per_cycle,
            "fp64_pipe_active_pct": num(rec, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": num(rec, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "registers": num(rec, "launch__registers_per_thread")}


def main():
    raw, key, cfg = sys.argv[1], sys.argv[2], sys.argv[3]
    out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "profiles", "r02", "ncu_flops.json")
    import bipb_inputs as g
    n = g.config(cfg).n
    recs = read_raw(raw)
    rec = max(recs, key=lambda r: num(r, "gpu__time_duration.sum"))  # the dominant launch
    s = summarise(rec, n * (n - 1))
    s["source"] = os.path.relpath(raw, ROOT)
    db = json.load(open(out)) if os.path.exists(out) else {}
    db[f"{key}_{cfg}"] = s
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump(db, open(out, "w"), indent=1)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
