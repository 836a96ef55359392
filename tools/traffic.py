"""DRAM traffic per launch class from an ncu capture
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
      --csv --log-file X.csv python bench.py --T 3 --steps 1 --warmup 0 ...
-> profiles/traffic_per_launch.json {class: {dram_bytes_per_unit, launches}}
(units: frame pixels H*W, or all N vertices for analyze / range).
python tools/traffic.py X.csv H W T"""
import collections
import csv
import json
import sys
from pathlib import Path

CLASSES = {  # kernel name prefix -> (bench launch class, counts as a launch)
    "vfcp::enc_block_kernel": ("enc_block", True),
    # the block scan of a frame: chain kernel + its dependent interior kernel
    "vfcp::bs_chain_kernel<1": ("bs_chain", True),
    "vfcp::bs_interior_kernel<1": ("bs_chain", False),
    "vfcp::cube_kernel": ("analyze", True), "vfcp::exact_kernel": ("analyze", True),
    "vfcp::analyze_kernel": ("analyze", True), "vfcp::range_kernel": ("range", True),
    # the decoder's block kernels of a frame: fast + general (listed blocks)
    "vfcp::dec_block_fast_kernel": ("dec_block", True),
    "vfcp::dec_block_kernel": ("dec_block", False),
    "vfcp::bs_chain_kernel<0": ("dec_chain", True),
    "vfcp::bs_interior_kernel<0": ("dec_chain", False),
}
UNIT = {"bytes": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}


def main(path, H, W, T):
    acc = collections.defaultdict(lambda: collections.defaultdict(float))
    launches = collections.defaultdict(set)
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].replace("void ", "").split("(")[0]
        cls, counts = next((c for k, c in CLASSES.items() if name.startswith(k)),
                           (None, False))
        if cls is None:
            continue
        m = d["Metric Name"]
        if m.startswith("dram__bytes"):
            acc[cls]["bytes"] += float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1)
            if counts:
                launches[cls].add(d["ID"])
    out = {}
    for cls, a in acc.items():
        n = len(launches[cls])
        if cls == "analyze":
            # one analysis = cube + exact + the (empty) fused fallback launch
            n = max(1, n // 3)
        units = H * W * T if cls in ("analyze", "range") else H * W
        out[cls] = {"dram_bytes_per_unit": round(a["bytes"] / n / units, 4),
                    "launches": n}
    dst = Path(__file__).resolve().parents[1] / "profiles" / "traffic_per_launch.json"
    dst.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
