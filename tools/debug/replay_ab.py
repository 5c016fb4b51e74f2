"""bench.py's replay section alone, per library variant (debug A/B):
    python tools/debug/replay_ab.py lib.so ...  (each in its own process)"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] != "--one":
    for rep in range(3):
        for lib in sys.argv[1:]:
            env = dict(os.environ, SPARROW_LIB_PATH=os.path.abspath(lib))
            out = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True,
                                 text=True, cwd=ROOT).stdout.strip().splitlines()
            print(os.path.basename(lib), out[-1] if out else "failed", flush=True)
    sys.exit(0)
sys.path.insert(0, ROOT)
import torch
import bench
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
clean = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
def flush_l2(k):
    flush.fill_(k & 0xFF)
    clean.sum()
r = bench.replay_bench(dev, flush_l2, 6536.4)
a = {x["rows_per_call"]: x for x in r["append"]}
print(json.dumps({"append4096_us": a[4096]["us"], "append65536_us": a[65536]["us"],
                  "stream_frac": a[65536]["stream"]["frac"], "stream_us": a[65536]["stream"]["us_per_call"]}))
