"""Print the key numbers of one tools/iter.sh run: python tools/show_iter.py TAG"""
import csv, json, subprocess, sys
tag = sys.argv[1]
for line in open(f"gpurun_out/{tag}_bench.log"):
    if line.startswith('{"metric'):
        d = json.loads(line)
        print("config2", round(d["ms_per_step"], 3), "ms/step", f"{d['value']:.3e}", d["stages_ms"])
try:
    for line in open(f"gpurun_out/{tag}_compose.log"):
        if line.startswith("{"):
            d = json.loads(line)
            print("compose", d["config"]["workload"][:48], f"{d['value']:.1f}", d["stages_ms"])
except FileNotFoundError:
    pass
try:
    out = subprocess.run(["ncu", "-i", f"gpurun_out/{tag}_ncu.ncu-rep", "--page", "details", "--csv"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    ik, im, iv, iu, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Executed Instructions",
            "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction"]
    for x in r[1:]:
        if x[im] in want:
            print(" ", x[iid], x[ik][:34], x[im], x[iv], x[iu])
except Exception as e:
    print("ncu:", e)
