import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "fps %.0f step %.4f ms fwd %.1f us (%.3f) bwd %.1f us (%.3f)" % (
            d["value"], d["ms_per_step"], d["kernel_ms"]["fwd"] * 1e3, d["roofline"]["fwd_kernel"]["frac"],
            d["kernel_ms"]["bwd"] * 1e3, d["roofline"]["frac"]))
    except Exception as e:
        print(f, "ERR", e)
