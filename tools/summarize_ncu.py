"""Turns the ncu raw-page CSV of one captured apply (tools/profile_fd.py --names-out) into the
per-launch table committed under profiles/ and the traffic map bench.py reads."""
import csv
import json
import sys

KEYS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dmma_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "warps": "sm__warps_active.avg.per_cycle_active",
    "regs": "launch__registers_per_thread",
    "block": "launch__block_size",
    "grid": "launch__grid_size",
    "sm_mhz": "smsp__cycles_elapsed.avg.per_second",
}


def main(raw_csv, names_json, out_md_rows, traffic_json, cfg):
    rows = list(csv.reader(open(raw_csv)))
    hdr, units = rows[0], rows[1]
    names = json.load(open(names_json))
    launches = names["launches"]
    data = rows[2:]
    assert len(data) == len(launches), (len(data), len(launches))
    table, traffic = [], {}
    for (nm, fl), r in zip(launches, data):
        g = {}
        for k, m in KEYS.items():
            i = hdr.index(m) if m in hdr else None
            g[k] = r[i] if i is not None else ""
            if i is not None and k in ("dram_read", "dram_write"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[i], 1)
                g[k] = float(r[i].replace(",", "")) * scale
            if i is not None and k == "dur_us":
                scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(units[i], 1)
                g[k] = float(r[i].replace(",", "")) * scale
        tb = g["dram_read"] + g["dram_write"]
        traffic[nm] = tb
        tf = fl / (g["dur_us"] * 1e-6) / 1e12 if fl else 0.0
        table.append(f"| {cfg} | {nm} | {r[hdr.index('Kernel Name')].split('(')[0].replace('void ', '')[-40:]} | "
                     f"{g['dur_us']:.1f} | {tf:.1f} | {g['dmma_pct']} | {g['dram_read'] / 1e6:.0f} / {g['dram_write'] / 1e6:.0f} | "
                     f"{tb / names['n_dof']:.1f} | {g['block']}x{g['grid']} | {g['regs']} |")
    tj = json.load(open(traffic_json)) if __import__("os").path.exists(traffic_json) else {}
    tj[cfg] = traffic
    json.dump(tj, open(traffic_json, "w"), indent=1)
    open(out_md_rows, "a").write("\n".join(table) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
