"""e2e (pinned host, 4-chunk budget) of the bench's gaussian + median step vs pipeline slot size."""
import os, subprocess, sys, json
for mb in ("160", "160", "320", "160"):
    env = dict(os.environ, HB_SLOT_MB=mb)
    out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "2", "--no-cpu", "--workload", "headline"],
                         env=env, capture_output=True, text=True).stdout
    line = [l for l in out.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    print(f"slot {mb} MiB: e2e {d['e2e']['value']} Gvox/s", flush=True)
