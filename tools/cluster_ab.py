"""Small-grid cluster path vs the multi-kernel path (kernel timing off):
  python tools/cluster_ab.py C1 C2"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = open(os.path.join(ROOT, "tools", "graph_ab.py")).read().split("CODE = r'''")[1].split("'''")[0]
for cfg in sys.argv[1:]:
    for mode, env in (("cluster", {}), ("multi-kernel", {"GS_NO_CLUSTER": "1"})):
        out = subprocess.run([sys.executable, "-c", CODE % (ROOT, cfg)], capture_output=True, text=True,
                             env={**os.environ, **env})
        try:
            print(cfg, mode, round(json.loads(out.stdout.strip().splitlines()[-1])["steps_per_s"], 1))
        except Exception:
            print(cfg, mode, "failed", out.stderr[-400:])
