"""One hash launch per BASELINE config, for a single `ncu --set full` capture
of every config's dominant kernel; then fold the capture into
profiles/ncu_summary.json keyed by the bench's config names (bench.py reads
roofline.traffic from it).

on the GPU box (one process, one GPU):
  ncu --set full --import-source on --clock-control none \
      -k regex:"k_fixed|k_varlen|k_generic|k_decimal" -o gpurun_out/ncu_cfg_<tag> \
      python tools/ncu_configs.py run gpurun_out/ncu_cfg_<tag>_order.json
  ncu -i gpurun_out/ncu_cfg_<tag>.ncu-rep --page raw --csv > gpurun_out/ncu_cfg_<tag>_raw.csv
here:
  python tools/ncu_configs.py fold <tag> gpurun_out/ncu_cfg_<tag>_raw.csv gpurun_out/ncu_cfg_<tag>_order.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(order_path, only=None):
    import torch

    import bench
    from paper_2407_09333_b200 import _native

    torch.cuda.set_device(0)
    bench.PROFILE_ONLY = True
    names = []
    specs = [("md5_1k", bench.WORKLOADS["md5_1k"])] + bench.suite_specs()
    for name, spec in specs:
        if only and name not in only:
            continue
        w = bench.make_workload(name, spec, 0, 0, 0, 1)
        w.free_extra()
        torch.cuda.synchronize()
        w.step() if w.kind != "fixed" else w.probe_kernel()
        torch.cuda.synchronize()
        names.append({"config": name, "kernel": _native.last_kernel_name(), "alg_bytes": w.alg_bytes})
        print(name, names[-1]["kernel"][:80], flush=True)
        del w
        torch.cuda.empty_cache()
    with open(order_path, "w") as f:
        json.dump(names, f, indent=1)


def fold(tag, raw_csv, order_path):
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from ncu_summary import raw, to_bytes

    rows = raw(raw_csv)
    order = json.load(open(order_path))
    if len(rows) != len(order):
        raise SystemExit(f"{len(rows)} profiled kernels vs {len(order)} configs")
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(p)) if os.path.exists(p) else {}
    md = [f"# ncu --set full, one launch per BASELINE config ({tag})", "",
          "dram bytes = dram__bytes_read.sum + dram__bytes_write.sum of the config's hash kernel; "
          "algorithmic = message bytes read once + digests (+ offsets) written once.", "",
          "| config | kernel | ms | dram GB | algorithmic GB | traffic / alg | ALU % | FMA % | issue % | DRAM % |",
          "|---|---|---|---|---|---|---|---|---|---|"]
    for r, o in zip(rows, order):
        def val(k):
            v = r.get(k)
            return to_bytes(*v) if v else None
        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        dram = (rd or 0) + (wr or 0)
        rec = {"kernel": r["Kernel Name"][0], "dram_bytes": dram, "duration_ms": val("gpu__time_duration.sum") / 1e6
               if r.get("gpu__time_duration.sum", ("", ""))[1] in ("nsecond", "ns") else val("gpu__time_duration.sum"),
               "alu_pipe_pct": val("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
               "fma_pipe_pct": val("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
               "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
               "dram_pct": val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
               "warp_instructions": val("smsp__inst_executed.sum"),
               "algorithmic_bytes": o["alg_bytes"], "traffic_over_algorithmic": round(dram / o["alg_bytes"], 4),
               "source": f"{os.path.basename(raw_csv)} ({tag})"}
        summ[o["config"]] = rec
        md.append(f"| {o['config']} | `{rec['kernel'].split('(')[0]}` | {rec['duration_ms']:.4f} | "
                  f"{dram / 1e9:.4f} | {o['alg_bytes'] / 1e9:.4f} | {rec['traffic_over_algorithmic']:.4f} | "
                  f"{rec['alu_pipe_pct']:.1f} | {rec['fma_pipe_pct']:.1f} | {rec['issue_active_pct']:.1f} | "
                  f"{rec['dram_pct']:.1f} |")
    with open(p, "w") as f:
        json.dump(summ, f, indent=1)
    with open(os.path.join(ROOT, "profiles", f"ncu_configs_{tag}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], set(sys.argv[3:]) or None)
    else:
        fold(sys.argv[2], sys.argv[3], sys.argv[4])
