"""DRAM traffic per kernel from an ncu --set full report -> JSON (bench.py's roofline.traffic).

    python tools/ncu_traffic.py gpurun_out/rNN/prof_full.ncu-rep SLICES > profiles/rNN/ncu_traffic.json
SLICES: slices per launch in the captured command (bench.py --slices).
"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, slices):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    res = {}
    for r in rows[2:]:
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("bsct::", "")
        rd = float(r[ix["dram__bytes_read.sum"]].replace(",", "")) * UNIT[units[ix["dram__bytes_read.sum"]]]
        wr = float(r[ix["dram__bytes_write.sum"]].replace(",", "")) * UNIT[units[ix["dram__bytes_write.sum"]]]
        res[name.split("<")[0]] = {"kernel": name, "dram_read_bytes": rd, "dram_write_bytes": wr,
                                   "slices_per_launch": slices, "bytes_per_slice": (rd + wr) / slices}
    json.dump({"source": path, "note": "ncu --set full, one launch per kernel; writes still resident in L2 at "
                                      "kernel end are not counted", "kernels": res}, sys.stdout, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
