"""Summarize tools/ncu_multi.py captures (one rank, single-pass metric sets):
per kernel launch of the op list, device duration, DRAM read+write bytes and
NVLink tx/rx bytes next to the op's algorithmic bytes."""

import csv
import json
import sys

MIB = 1 << 20


def rows(path):
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    out = list(csv.DictReader(lines[start:]))
    return [r for r in out if r.get("ID", "").isdigit()]


def algo_bytes(tag, op, nbytes, p):
    if op == "all_reduce":
        bus = 2 * (p - 1) / p * nbytes
    elif op == "all_to_all_single":
        bus = (p - 1) / p * nbytes
    else:
        bus = nbytes
    return bus


def main(dram_csv, nvl_csv, world, out_json):
    from ncu_multi import OPS  # noqa: E402  (same op list, same order)

    d, n = rows(dram_csv), rows(nvl_csv)
    reps = len(d) // len(OPS)
    table = []
    for i, (tag, op, nbytes, algo) in enumerate(OPS):
        for k in range(reps):
            a, b = d[i * reps + k], n[i * reps + k]
            t_ns = float(a["gpu__time_duration.sum"])
            dram = float(a["dram__bytes_read.sum"]) + float(a["dram__bytes_write.sum"])
            bus = algo_bytes(tag, op, nbytes, world)
            table.append({
                "op": tag, "kernel": a["Kernel Name"].split("(")[0].replace("void ", ""),
                "grid": a["Grid Size"], "duration_us": round(t_ns / 1e3, 2),
                "bus_bytes": int(bus), "busbw_gbs": round(bus / t_ns, 1),
                "dram_bytes": int(dram), "dram_gbs": round(dram / t_ns, 1),
                "nvltx_bytes": int(float(b["nvltx__bytes.sum"])),
                "nvlrx_bytes": int(float(b["nvlrx__bytes.sum"])),
                "nvltx_gbs": round(float(b["nvltx__bytes.sum"]) / float(b.get("gpu__time_duration.sum") or t_ns), 1)
                if b.get("gpu__time_duration.sum") else round(float(b["nvltx__bytes.sum"]) / t_ns, 1),
            })
    json.dump({"world": world, "rank_profiled": 0, "method": "ncu single-pass metric sets on one "
               "rank of a live multi-rank run (tools/ncu_multi.py), cold-ish serialized launches",
               "launches": table}, open(out_json, "w"), indent=1)
    print(f"p = {world}")
    for r in table:
        print(f"  {r['op']:22s} {r['kernel']:38s} {r['duration_us']:9.1f} us  bus {r['busbw_gbs']:7.1f} GB/s"
              f"  dram {r['dram_bytes'] / MIB:9.1f} MiB  nvl tx/rx {r['nvltx_bytes'] / MIB:8.1f}/{r['nvlrx_bytes'] / MIB:8.1f} MiB")


if __name__ == "__main__":
    sys.path.insert(0, __import__("os").path.dirname(__file__))
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4])
