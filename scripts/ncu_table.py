"""Print selected ncu raw metrics of a report as a compact table:
    python scripts/ncu_table.py REPORT.ncu-rep metric1 metric2 ..."""
import csv
import io
import subprocess
import sys

rep, metrics = sys.argv[1], sys.argv[2:]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
metrics = [m for m in metrics if m in hdr]
idx = [hdr.index(m) for m in metrics]
short = [m.split("__")[-1][:22] for m in metrics]
print("kernel".ljust(28), " ".join(s.rjust(22) for s in short))
print("".ljust(28), " ".join(units[i].rjust(22) for i in idx))
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")[:28]
    print(name.ljust(28), " ".join(r[i].rjust(22) for i in idx))
