import sys, os, json
sys.path.insert(0, "/root/repo")
sys.argv = [sys.argv[0]]
import tools.bench_all as BA
for prec in ("c128", "c64"):
    r = BA.run("cfg3", prec, 1024)
    print(os.environ.get("HQ_TILE_BITS", "-"), json.dumps({k: r[k] for k in ("precision", "ms_per_step", "samples_per_s", "plan")})[:300], flush=True)
