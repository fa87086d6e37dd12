"""Fold one tools/gpu_full.sh pass (gpurun_out/*_<TAG>*) into profiles/.

usage: python tools/collect_evidence.py <TAG> <old profiles dir> <new profiles dir>
       e.g. python tools/collect_evidence.py r1v11 r1_v10 r1_v11

Moves profiles/<old>/ to profiles/<new>/ (git mv: files not re-measured, such
as e2e_pageable.txt or runtime_bench.txt, keep their history), overwrites the
bench lines, GPU/pytest/smoke logs, launch list and configs with the new
pass, regenerates profiles/sweep_r1.md, the stall breakdown and the ncu
summary (profiles/ncu_<new>.md + ncu_summary.json).
"""
import glob
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
WORKLOADS = ["sha1_64", "sm3_1k", "sha1_1k", "varlen_md5", "varlen_sha1", "varlen_sm3", "paper_sha1", "paper_md5",
             "paper_sm3"]
NCU = ["md5_1k", "sha1_1k", "sm3_1k", "varlen_md5", "paper_md5"]


def run(*cmd, **kw):
    return subprocess.run(cmd, cwd=ROOT, check=True, **kw)


def main():
    tag, old, new = sys.argv[1:4]
    src, dst = os.path.join(ROOT, "profiles", old), os.path.join(ROOT, "profiles", new)
    if os.path.isdir(src) and not os.path.isdir(dst):
        run("git", "mv", src, dst)
    os.makedirs(dst, exist_ok=True)
    stale = set(glob.glob(os.path.join(dst, "gpu_r1v*.txt")) + glob.glob(os.path.join(dst, "pytest_gpu_*.log")) +
                glob.glob(os.path.join(dst, "smoke_*.log")) + glob.glob(os.path.join(dst, "*_final.*")))
    for f in sorted(stale):
        run("git", "rm", "-q", "-f", "--ignore-unmatch", f)
        if os.path.exists(f):
            os.remove(f)
    shutil.copy(os.path.join(OUT, f"bench_{tag}.json"), os.path.join(dst, "bench.json"))
    shutil.copy(os.path.join(OUT, f"bench_ref_{tag}.json"), os.path.join(dst, "bench_ref.json"))
    for w in WORKLOADS:
        shutil.copy(os.path.join(OUT, f"bench_{w}_{tag}.json"), os.path.join(dst, f"bench_{w}.json"))
    for name in (f"gpu_{tag}.txt", f"pytest_gpu_{tag}.log", f"smoke_{tag}.log"):
        shutil.copy(os.path.join(OUT, name), os.path.join(dst, name))
    shutil.copy(os.path.join(OUT, f"launches_{tag}.csv"), os.path.join(dst, "launches.csv"))
    shutil.copy(os.path.join(OUT, f"configs_{tag}.jsonl"), os.path.join(dst, "configs.jsonl"))
    table = subprocess.run([sys.executable, "tools/sweep_table.py", os.path.join(dst, "configs.jsonl")], cwd=ROOT,
                           check=True, capture_output=True, text=True).stdout
    table = table.replace("(configs.jsonl)", f"({new}: profiles/{new}/configs.jsonl)")
    with open(os.path.join(ROOT, "profiles", "sweep_r1.md"), "w") as f:
        f.write(table)
    stalls = []
    for w in NCU:
        src_csv = os.path.join(OUT, f"source_{w}_{tag}.csv")
        if os.path.exists(src_csv):
            stalls.append(subprocess.run([sys.executable, "tools/stall_summary.py", src_csv, "--top", "6"], cwd=ROOT,
                                         capture_output=True, text=True).stdout)
    with open(os.path.join(dst, "stalls.txt"), "w") as f:
        f.write("".join(stalls))
    raws = [os.path.join(OUT, f"raw_{w}_{tag}.csv") for w in NCU if os.path.exists(os.path.join(OUT, f"raw_{w}_{tag}.csv"))]
    run(sys.executable, "tools/ncu_summary.py", new, *raws, "--launches", os.path.join(OUT, f"launches_{tag}.csv"),
        stdout=subprocess.DEVNULL)
    print(f"profiles/{new} updated from {tag}")


if __name__ == "__main__":
    main()
