"""Turn an ncu --set full report of profiles/codec_probe.py into
profiles/traffic.json: DRAM bytes (read + write) per launch of every codec
kernel on one full Llama-3.1-8B chunk (T = 8192). bench.py reports it as
the dominant kernel's `traffic` next to the algorithmic bytes.

  python profiles/ncu_traffic.py gpurun_out/<report>.ncu-rep > profiles/traffic.json
"""
import csv
import io
import json
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
ki, rd, wr = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
acc = {}
for r in rows[2:]:
    name = r[ki].split("(")[0].replace("void ", "").strip()
    b = float(r[rd].replace(",", "")) * scale[units[rd]] + float(r[wr].replace(",", "")) * scale[units[wr]]
    acc.setdefault(name, []).append(b)
out = {k: int(sum(v) / len(v)) for k, v in acc.items()}
print(json.dumps(out, indent=1, sort_keys=True))
