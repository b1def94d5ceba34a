"""Summarise a SPECEDGE_PARITY_LOG jsonl (tests/gpu_helpers.py) as the markdown tables of
profiles/rNN_parity_stats.md.  Usage: python tools/parity_stats.py LOG.jsonl "title" > OUT.md"""
import json
import sys


def main(path, title):
    rows = [json.loads(l) for l in open(path) if l.strip()]
    name = lambda r: r["test"].split("::")[-1]
    f = lambda x: "nan" if x is None else f"{x:.4f}"
    print(f"# {title}\n")
    print("Contract: `tests/gpu_helpers.py` (DESIGN.md §4 R-tolerances).  `bound` = the max-abs logit bound the")
    print("test applied: 2e-2, or 2 × the oracle's own fp32-level deviation (`noise_max`) where larger.\n")
    print("## Logits (GPU fp32 capture of the LM head vs oracle float64)\n")
    print("| test | logits | max | q99.9 | q99 | oracle noise max | bound |")
    print("|---|---|---|---|---|---|---|")
    for r in rows:
        if r["kind"] == "logits":
            print(f"| {name(r)} | {r['n']} | {f(r['gpu_max'])} | {f(r['gpu_q999'])} | {f(r['gpu_q99'])} | "
                  f"{f(r.get('noise_max'))} | {f(r['bound'])} |")
    print("\n## Acceptance (oracle-margin exemptions)\n")
    print("| test | requests | exempt | requests whose oracle path visits a margin <= 1e-2 | slots | "
          "slots with margin <= 1e-2 |")
    print("|---|---|---|---|---|---|")
    tot = [0, 0]
    for r in rows:
        if r["kind"] == "acceptance":
            tot[0] += r["requests"]
            tot[1] += r["exempt"]
            print(f"| {name(r)} | {r['requests']} | {r['exempt']} | {r['low_margin_paths']} | {r['slots']} | "
                  f"{r['low_margin_slots']} |")
    print(f"\nTotal: {tot[0]} requests checked, {tot[1]} exempt.")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "Parity statistics")
