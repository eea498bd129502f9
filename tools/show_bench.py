import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d["kernel_ms"]
        main = k.get("bwd_main")
        print(f, "fps %.0f step %.4f ms fwd %.1f us (%.3f) bwd %.1f us%s (frac %.3f)" % (
            d["value"], d["ms_per_step"], k["fwd"] * 1e3, d["roofline"]["fwd_kernel"]["frac"],
            k["bwd"] * 1e3, (" [main %.1f + fin %.1f]" % (main * 1e3, k["bwd_finish"] * 1e3)) if main else "",
            d["roofline"]["frac"]))
    except Exception as e:
        print(f, "ERR", e)
