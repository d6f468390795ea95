import sys, json
sys.path.insert(0, "/root/repo")
import bench
hbm, _ = bench.peaks()
for tw in [int(x) for x in sys.argv[1:]]:
    bench.CONFIGS["c5"]["tile_width"] = tw
    r = bench.side_config_bench("c5", hbm)
    print(tw, json.dumps({k: r[k] for k in ("tile_width", "format", "us", "alg_bytes", "frac_hbm")}), flush=True)
