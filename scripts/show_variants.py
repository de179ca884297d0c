import glob, json, sys
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/v_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{f:50s} step {d['ms_per_step']:9.3f}  last {d['phases_ms']['last_node_total']:9.3f}  "
              f"frac {d['roofline']['frac']:.3f}  {d['result']['count']} {d['result']['checksum']}")
    except Exception as e:
        print(f, "ERR", e)
