"""Write profiles/ncu_traffic.json from an ncu report (--set full, or just the
dram__bytes_read/write metrics) of `bench.py --steps 1 --warmup 3 [--nz NZ]
--no-e2e --no-cpu-baseline` (the bench workload, or the same CTA / tile /
z-chunk structure with NZ z layers): DRAM bytes per launch of the tiled3d
kernels, per cell, scaled to the bench's 512 x 512 x 256 grid.  bench.py reads `pre_dram_bytes_per_launch`
for the roofline line's `traffic`.
Usage: python tools/ncu_traffic.py REPORT.ncu-rep NZ"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# algorithmic bytes per cell and launch: V_z pressure launch
# reads 1 source + p read/write; merged V_x+V_y reads 2 sources + p; velocity
# reads p + 3 v read/write
ALG = {"tiled3d<3, 1>": 1536, "tiled3d<3, 2>": 2048, "tiled3d<3, 3>": 3584}


def main(path, nz):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    name_i = hdr.index("Kernel Name")
    cells = 512 * 512 * nz
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    launches = []
    for r in rows[2:]:
        name = r[name_i]
        key = next((k for k in ALG if k in name), None)
        if key is None:
            continue
        rd = float(r[hdr.index("dram__bytes_read.sum")]) * scale[units[hdr.index("dram__bytes_read.sum")]]
        wr = float(r[hdr.index("dram__bytes_write.sum")]) * scale[units[hdr.index("dram__bytes_write.sum")]]
        launches.append({"kernel": name[:60], "dram_read": rd, "dram_write": wr,
                         "bytes_per_cell": (rd + wr) / cells, "algorithmic_bytes_per_cell": ALG[key],
                         "duration_unit": units[hdr.index("gpu__time_duration.sum")],
                         "duration": float(r[hdr.index("gpu__time_duration.sum")])})
    pre = [l["bytes_per_cell"] for l in launches if "<3, 1>" in l["kernel"]]
    vel = [l["bytes_per_cell"] for l in launches if "<3, 3>" in l["kernel"]]
    res = {"source": f"ncu --set full of `bench.py --steps 1 --warmup 3 --nz {nz}` (the bench workload with {nz} "
                     "instead of 256 z layers per GPU; identical CTA/tile/z-chunk structure); per-cell bytes "
                     "scaled to 512x512x256",
           "launches": launches}
    if pre:
        res["pre_bytes_per_cell"] = sum(pre) / len(pre)
        res["pre_dram_bytes_per_launch"] = res["pre_bytes_per_cell"] * 512 * 512 * 256
    if vel:
        res["vel_bytes_per_cell"] = sum(vel) / len(vel)
        res["vel_dram_bytes_per_launch"] = res["vel_bytes_per_cell"] * 512 * 512 * 256
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
