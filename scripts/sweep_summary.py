import json, sys
for l in open(sys.argv[1]):
    l = l.strip()
    if l.startswith('{"config"'):
        d = json.loads(l)
        print(d["config"], d["env"], "fmt", d["format"], "sch", d["schedule"], "us", [round(u) for u in d["us"]],
              "GBps", [round(g) for g in d["GBps"]], "frac %.3f / 88n %.3f" % (d["iter_frac"], d["iter_frac_vs_88n"]),
              "solve", d.get("solve_s"), d.get("iterations"))
    elif l and not l.startswith("{"):
        print(l[:200])
