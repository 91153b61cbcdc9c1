"""Build profiles/ncu_traffic.json (per-phase DRAM bytes per launch) from an ncu launch list
(`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`) of ONE bench
step (`bench.py --steps 1 --warmup 0`): the second occurrence of each kernel is the timed step."""
import csv
import hashlib
import json
import os
import sys
import time

PHASE = {"k_relax_first": "watershed.init", "k_relax_round": "watershed.relax", "k_resolve": "watershed.select",
         "k_jump": "watershed.jump", "k_jumpv": "watershed.jump", "k_union": "watershed.union", "k_root_merge": "watershed.find",
         "k_root_label": "watershed.find", "k_root_store": "watershed.find", "k_relabel": "watershed.relabel", "k_relabel4": "watershed.relabel", "k_root_canon": "watershed.find",
         "k_compress_pairs": "watershed.union",
         "k_dense": "waterfall.dense_ids", "k_dimage": "waterfall.dense_ids", "k_dimage_rk": "waterfall.dense_ids",
         "k_tile_list": "watershed.relax", "k_union_pairs": "watershed.union", "k_grad_fused": "gradient.fused", "k_rag": "waterfall.rag", "k_edges": "waterfall.levels",
         "k_hook": "waterfall.levels", "k_flatten": "waterfall.levels", "k_levelmap": "waterfall.levels",
         "k_iota": "waterfall.levels", "k_levels": "waterfall.materialise", "k_blur_axis": "gradient.blur",
         "k_gradmag": "gradient.magnitude", "k_grad_stream": "gradient.fused",
         "k_relabel_seg": "watershed.relabel", "k_root_bits": "waterfall.dense_ids", "k_rank_sum": "waterfall.dense_ids",
         "k_scan_counts": "waterfall.dense_ids", "k_rank_write": "waterfall.dense_ids",
         "k_root_dense": "waterfall.dense_ids", "k_collect_roots": "watershed.jump",
         "k_e16_live": "waterfall.levels", "k_e16_lo": "waterfall.levels", "k_hook16": "waterfall.levels"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3,
        "msecond": 1, "ms": 1}


def main(path, out, n_vox):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ii, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
    launches = {}
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].split("<")[0].split("::")[-1].strip()
        if name.startswith("void "):
            name = name[5:]
        d = launches.setdefault(int(r[ii]), {"name": name})
        d[r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
    per = {}
    for lid in sorted(launches):
        d = launches[lid]
        ph = PHASE.get(d["name"])
        if not ph:
            continue
        p = per.setdefault(ph, {"launches": 0, "bytes": 0.0, "ms": 0.0, "kernels": set()})
        p["launches"] += 1
        p["bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        p["ms"] += d.get("gpu__time_duration.sum", 0)
        p["kernels"].add(d["name"])
    res = {}
    for ph, p in per.items():
        res[ph] = {"bytes_per_launch": p["bytes"] / p["launches"], "launches": p["launches"],
                   "ms_total_ncu": p["ms"], "kernels": sorted(p["kernels"]),
                   "note": "ncu cold-cache serialised; one bench step (--steps 1 --warmup 0) incl. its gradient pre-pass"}
    # the whole step: every watershed / waterfall launch of the ONE captured step
    step = sum(p["bytes"] for ph, p in per.items() if ph.startswith(("watershed.", "waterfall.")))
    step_ms = sum(p["ms"] for ph, p in per.items() if ph.startswith(("watershed.", "waterfall.")))
    lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2410_08946_b200",
                       "libws_b200.so")
    res["_step"] = {"dram_bytes": step, "ms_ncu": step_ms, "voxels": n_vox,
                    "dram_bytes_per_voxel": step / n_vox if n_vox else None,
                    "amplification_vs_38B": step / n_vox / 38.0 if n_vox else None}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hs = hashlib.sha256()
    for fn in sorted(__import__("glob").glob(os.path.join(root, "paper_2410_08946_b200", "csrc", "*"))) + \
            [os.path.join(root, "include", "ws.h")]:
        hs.update(os.path.basename(fn).encode())
        hs.update(open(fn, "rb").read())
    res["_provenance"] = {"src_sha256": hs.hexdigest(),
                          "lib_sha256": hashlib.sha256(open(lib, "rb").read()).hexdigest() if os.path.exists(lib) else None,
                          "launch_list": os.path.basename(path), "captured": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    json.dump(res, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(res, indent=1, sort_keys=True)[:3000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 805306368)
