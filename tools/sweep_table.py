"""Render the configs[4] sweep (bench_configs.py JSON lines) as markdown:
roofline fraction and GB/s per (algorithm, batch count, message size).

usage: python tools/sweep_table.py configs.jsonl > profiles/sweep_<tag>.md
"""
import json
import sys
from collections import defaultdict


def main():
    rows = [json.loads(ln) for ln in open(sys.argv[1]) if ln.startswith("{")]
    sw = [r for r in rows if r["config"] == "C5"]
    other = [r for r in rows if r["config"] != "C5"]
    print(f"# BASELINE configs on 1 B200 ({sys.argv[1].split('/')[-1]})\n")
    print("Kernel-only, inputs resident in HBM and read from HBM at every timed pass (batches under 2 x L2: "
          "10-copy graph replays with the L2 flushed before each; larger: back-to-back launches; launches flagged "
          "HB_FLAG_INPUT_READY as in bench.py, so consecutive passes overlap), CUDA events; every point's "
          "digests checked against a CPU reference on a row sample (`bit_exact_sample`). Fraction = "
          "max(T_hbm, T_alu, T_chain) / T_measured with T_hbm at the HBM peak (6,650 GB/s fallback unless "
          "MEASURED_PEAKS.json), T_alu = blocks x ALU-only ops / (64 lanes/clk x 148 SMs x clock) and "
          "T_chain = blocks per message x the measured dependent-chain latency of one compression "
          "(MD5 1,044 / SHA-1 1,116 / SM3 2,514 cycles, one warp per SM) -- the bound when the batch has too "
          "few messages to overlap; it is left out where consecutive flagged passes overlap on the GPU "
          "(`chain_applies`: false -- rows of <= 128 B, messages of <= 17 blocks, grids of >= one CTA per SM), "
          "since several batches' chains then run side by side.\n")
    print("| config | alg | messages | size | ms | GB/s | Mhash/s | bound | fraction | bit-exact |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in other:
        size = r.get("msg_len", r.get("len"))
        print(f"| {r['config']} | {r['alg']} | {r['n']} | {size} | {r['ms']} | {r['GBps']} | {r['Mhash_s']} | "
              f"{r['roofline']['bound']} | {r['roofline']['frac']:.2f} | {r['bit_exact_sample']} |")
    if not sw:
        return
    print("\n## configs[4] sweep: roofline fraction (GB/s below)\n")
    t = defaultdict(dict)
    for r in sw:
        t[(r["alg"], r["n"])][r["msg_len"]] = r
    Ls = sorted({r["msg_len"] for r in sw})
    print("| alg | messages | " + " | ".join(f"{L} B" for L in Ls) + " |")
    print("|---|---|" + "---|" * len(Ls))
    for k in sorted(t):
        print(f"| {k[0]} | {k[1]} | " + " | ".join(
            f"{t[k][L]['roofline']['frac']:.2f}" if L in t[k] else "" for L in Ls) + " |")
    print("\n| alg | messages | " + " | ".join(f"{L} B" for L in Ls) + " |")
    print("|---|---|" + "---|" * len(Ls))
    for k in sorted(t):
        print(f"| {k[0]} | {k[1]} | " + " | ".join(f"{t[k][L]['GBps']:.0f}" if L in t[k] else "" for L in Ls) + " |")
    bad = [r for r in sw if not r["bit_exact_sample"]]
    print(f"\n{len(sw)} sweep points, {len(sw) - len(bad)} bit-exact on the sampled rows.")


if __name__ == "__main__":
    main()
