"""Build profiles/ncu_summary.json from a round's ncu --set full captures.
Usage: python tools/ncu_json.py DIR [round-tag] [prefix]
Each <prefix><cfg>.ncu-rep (default prefix full_) is one launch of the config's STP kernel; the
elements of the launch are its grid size (one CTA per element: every tuned kernel) unless the
config is in ELEMS.  The per-element DRAM traffic feeds bench.py's roofline.traffic."""
import csv
import io
import json
import os
import subprocess
import sys

ELEMS = {"c2": None, "c3": None, "c4": None, "n9": None}
KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma_pipe_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "shared_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "shared_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return dict(zip(hdr, vals)), dict(zip(hdr, units))


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]
    return float(v.replace(",", "")) * scale


def main(d, tag, prefix="full_"):
    out = {}
    for cfg, elems in ELEMS.items():
        rep = os.path.join(d, f"{prefix}{cfg}.ncu-rep")
        if not os.path.exists(rep):
            continue
        v, u = raw(rep)
        if elems is None:
            elems = int(float(v["launch__grid_size"].replace(",", "")))
        traffic = to_bytes(v["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) + \
            to_bytes(v["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        ent = {"kernel": v.get("Kernel Name", v.get("Function Name", "")), "elements_per_launch": elems,
               "dram_bytes_per_launch": traffic, "dram_bytes_per_element": traffic / elems}
        for k, m in KEYS.items():
            if m in v:
                try:
                    ent[k] = float(v[m].replace(",", ""))
                except ValueError:
                    ent[k] = v[m]
        ent["note"] = (f"round {tag}: ncu --set full --clock-control none, one launch of the bench.py "
                       "config after 3 warm-ups (cold caches, serialised); tools/gpu_ncu_full.sh")
        out[cfg] = ent
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                           "ncu_summary.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r01", sys.argv[3] if len(sys.argv) > 3 else "full_")
