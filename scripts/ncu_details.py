"""Text summary of an .ncu-rep (details page): 'section | metric | unit | value' lines plus
the rule texts. Usage: python scripts/ncu_details.py report.ncu-rep > profiles/.../x.txt"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ix = {n: h.index(n) for n in ("Kernel Name", "Block Size", "Grid Size", "Section Name", "Metric Name", "Metric Unit",
                              "Metric Value", "Rule Type", "Rule Description", "Estimated Speedup")}
last = None
for r in rows[1:]:
    kn = r[ix["Kernel Name"]]
    if kn != last:
        print(f"== {kn} grid {r[ix['Grid Size']]} block {r[ix['Block Size']]}")
        last = kn
    if r[ix["Metric Name"]]:
        print(f"{r[ix['Section Name']]} | {r[ix['Metric Name']]} | {r[ix['Metric Unit']]} | {r[ix['Metric Value']]}")
    elif r[ix["Rule Description"]]:
        print(f"{r[ix['Rule Type']]} | {r[ix['Rule Description']]} | est. speedup {r[ix['Estimated Speedup']]}")
