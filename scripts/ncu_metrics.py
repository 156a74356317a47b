"""Print selected raw ncu metrics of the kernels in an .ncu-rep (name regex, metric regex)."""
import csv, re, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
mre = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    if not re.search(kre, name):
        continue
    print("==", name[:60], "id", r[h.index("ID")])
    for i, m in enumerate(h):
        if mre is None or mre.search(m):
            print(f"   {m:80s} {r[i]:>20s} {units[i]}")
