import json, sys
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        print(line[:300]); continue
    d = json.loads(line)
    c = d["config"]
    print(c["workload"][:40], "ms/step=%.3f" % d["ms_per_step"], "val=%.3g" % d["value"], "e2e=%.3g" % d["e2e"]["value"],
          c.get("ranks"), c.get("pass1_steps"), c.get("rse"), "kern GB/s=%.0f share=%.2f" % (d["roofline"]["achieved"], d["roofline"]["share_of_step"] or 0), "launches", d["gpu_launches"])
