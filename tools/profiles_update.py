"""Copy the round's evidence from gpurun_out/ (tools/final_evidence.sh) into profiles/."""
import collections, csv, json, os, shutil, subprocess, sys

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(R, "gpurun_out"), os.path.join(R, "profiles")
last = lambda f: open(os.path.join(G, f)).read().strip().splitlines()[-1]
for n in (1, 2, 4):
    open(os.path.join(P, f"r01_bench_medium_n{n}.json"), "w").write(last(f"fe_n{n}.log") + "\n")
shutil.copy(os.path.join(P, "r01_bench_medium_n1.json"), os.path.join(P, "r01_bench_n1.json"))
shutil.copy(os.path.join(G, "fe_launches.csv"), os.path.join(P, "r01_launches_bench_n1.csv"))
shutil.copy(os.path.join(G, "fe_tests.log"), os.path.join(P, "r01_gpu_tests.log"))
shutil.copy(os.path.join(G, "fe_smoke.log"), os.path.join(P, "r01_smoke.log"))
summ = lambda rep: subprocess.run([sys.executable, os.path.join(R, "tools", "ncu_summary.py"), os.path.join(G, rep)],
                                  capture_output=True, text=True).stdout
for rep, out in (("fe_passes.ncu-rep", "r01_ncu_passes_summary.txt"), ("fe_sweeps.ncu-rep", "r01_ncu_pc2_sweeps_summary.txt")):
    old = open(os.path.join(P, out)).read()
    notes = old[old.index("# Reading"):] if "# Reading" in old else ""
    open(os.path.join(P, out), "w").write(summ(rep) + "\n" + notes)
rows = list(csv.reader(open(os.path.join(P, "r01_launches_bench_n1.csv"))))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr, body = rows[hi], rows[hi + 1:]
kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(list)
for r in body:
    if len(r) > mv:
        agg[r[kn].split("(")[0]].append(float(r[mv]) / 1000)
tot = sum(sum(v) for v in agg.values())
b = json.loads(open(os.path.join(P, "r01_bench_n1.json")).read())
ra, rb = b["roofline"]["pass_a"]["ms"] * 1e3, b["roofline"]["pass_b"]["ms"] * 1e3
lines = ["# Round 1 — ncu launch list of `python bench.py --steps 3 --warmup 3` (1 GPU)", "",
         "Command: `ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 400 --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e`",
         "(launches 30000-30399 = inside the PCG loop of a warm solve; cold-cache, serialised: compare shares, not absolutes).", "",
         "| kernel | launches | mean us | share |", "|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")
lines += ["", "The PC1 loop is exactly these two kernels per iteration (no other launches in the loop).",
          f"Bench (`profiles/r01_bench_n1.json`, live in-solve durations, same command without ncu): pass A {ra:.1f} us, pass B {rb:.1f} us",
          f"-> pass B share {100 * rb / (ra + rb):.0f}% (ncu {100 * sum(agg['k_pass_b_pc1']) / tot:.0f}%).",
          f"Bench clocks: median SM {b['clocks']['sm_mhz']:.0f} MHz (max {b['clocks']['sm_max_mhz']:.0f}), reasons {b['clocks']['reasons']}."]
open(os.path.join(P, "r01_launches_summary.md"), "w").write("\n".join(lines) + "\n")
print(open(os.path.join(G, "fe_tests.log")).read().strip().splitlines()[-1])
print({n: json.loads(open(os.path.join(P, f"r01_bench_medium_n{n}.json")).read())["value"] for n in (1, 2, 4)})
