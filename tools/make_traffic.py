"""Build profiles/ncu_traffic.json (per-phase DRAM bytes per launch) from an ncu launch list
(`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`) of ONE bench
step (`bench.py --steps 1 --warmup 0`): the second occurrence of each kernel is the timed step."""
import csv
import json
import sys

PHASE = {"k_relax_first": "watershed.init", "k_relax_round": "watershed.relax", "k_resolve": "watershed.select",
         "k_jump": "watershed.jump", "k_union": "watershed.union", "k_root_merge": "watershed.find",
         "k_root_label": "watershed.find", "k_root_store": "watershed.find", "k_relabel": "watershed.relabel", "k_relabel4": "watershed.relabel", "k_root_canon": "watershed.find",
         "k_compress_pairs": "watershed.union",
         "k_dense": "waterfall.dense_ids", "k_dimage": "waterfall.dense_ids", "k_dimage_rk": "waterfall.dense_ids",
         "k_tile_list": "watershed.relax", "k_union_pairs": "watershed.union", "k_grad_fused": "gradient.fused", "k_rag": "waterfall.rag", "k_edges": "waterfall.levels",
         "k_hook": "waterfall.levels", "k_flatten": "waterfall.levels", "k_levelmap": "waterfall.levels",
         "k_iota": "waterfall.levels", "k_levels": "waterfall.materialise", "k_blur_axis": "gradient.blur",
         "k_gradmag": "gradient.magnitude"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3,
        "msecond": 1, "ms": 1}


def main(path, out):
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
    json.dump(res, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(res, indent=1, sort_keys=True)[:3000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
