#!/usr/bin/env python
"""Per-template-family SASS evidence from the in-tree cubin cache (no GPU needed).

For every kernel family (korch_gemm / korch_pgemm / korch_attn / korch_conv ... and the
SIMT row-template families korch_pw / korch_rr / korch_cr / korch_tr) disassemble up to
N kernels with `cuobjdump -sass` and count the instructions that prove the sm_100a
paths: UTC*MMA (tcgen05.mma), UTMALDG (TMA tensor loads), LDTM (tcgen05.ld), UTMACCTL /
UTCBAR (tensor-map prefetch, tcgen05.commit), SYNCS (mbarrier), LDG.E.128 / STG.E.128
(128-bit global accesses), SHFL (warp shuffles).  Writes a JSON summary.

    python tools/sass_counts.py [--per-family 4] [--out profiles/r02_sass_counts.json]
"""
import argparse
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CACHE = os.path.join(ROOT, "paper_2406_09465_b200", "kcache")
PATTERNS = {
    "UTCxMMA (tcgen05.mma)": r"\bUTC\w*MMA\b",
    "UTMALDG (TMA load)": r"\bUTMALDG\b",
    "UTMASTG (TMA store)": r"\bUTMASTG\b",
    "LDTM (tcgen05.ld)": r"\bLDTM\b",
    "UTCBAR (tcgen05.commit)": r"\bUTCBAR\b",
    "SYNCS (mbarrier)": r"\bSYNCS\b",
    "LDG.128": r"\bLDG\.E\.(?:EL\.|CONSTANT\.)*128\b|\bLDG\.E\.128\b|\bLDG\.E\.\S*128",
    "STG.128": r"\bSTG\.E\.\S*128|\bSTG\.E\.128\b",
    "SHFL": r"\bSHFL\b",
    "ACQBULK/UBLKCP (bulk copy)": r"\bUBLKCP\b",
    "UTMALDG multicast": r"\bUTMALDG\S*MULTICAST",
    "STAS (st.async, DSMEM + mbarrier)": r"\bSTAS\b",
    "UCGABAR (cluster barrier)": r"\bUCGABAR_\w+",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--per-family", type=int, default=4)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sass_counts.json"))
    a = ap.parse_args()
    fams = collections.defaultdict(list)
    for f in sorted(os.listdir(CACHE)):
        if f.endswith(".ref"):
            name = f.split(".")[0]
            fam = name.rsplit("_", 1)[0]
            fams[fam].append((name, open(os.path.join(CACHE, f)).read().strip()))
    out = {"cache": os.path.relpath(CACHE, ROOT), "families": {}}
    for fam, ks in sorted(fams.items()):
        rows = []
        for name, cub in ks[: a.per_family]:
            sass = subprocess.run(["cuobjdump", "-sass", "-fun", name, os.path.join(CACHE, cub)],
                                  capture_output=True, text=True).stdout
            arch = re.search(r"arch = (sm_\w+)", sass)
            cnt = {k: len(re.findall(p, sass)) for k, p in PATTERNS.items()}
            cnt = {k: v for k, v in cnt.items() if v}
            rows.append({"kernel": name, "arch": arch.group(1) if arch else None,
                         "instructions": sum(1 for ln in sass.splitlines() if re.match(r"\s+/\*[0-9a-f]{4}\*/", ln)),
                         "counts": cnt})
        out["families"][fam] = {"kernels_in_cache": len(ks), "sampled": rows}
        tot = collections.Counter()
        for r in rows:
            tot.update(r["counts"])
        print(f"{fam:14s} {len(ks):5d} kernels  " + ", ".join(f"{k.split()[0]} {v}" for k, v in sorted(tot.items())))
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
