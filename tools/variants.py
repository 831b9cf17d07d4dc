"""Build libqtsse variants with extra -D flags (experiments): python tools/variants.py name=-DFOO=1,-DBAR ...
Outputs variants/<name>.so; on the GPU box swap one in for paper_1912_10024_b200/libqtsse.so."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_10024_b200 import build as B

os.makedirs(B.ROOT / "variants", exist_ok=True)
t = B.TARGETS["libqtsse"]
for arg in sys.argv[1:]:
    name, _, flags = arg.partition("=")
    out = B.ROOT / "variants" / f"{name}.so"
    cmd = t["cmd"](t["srcs"], out)
    cmd[1:1] = [f for f in flags.split(",") if f]
    r = subprocess.run(cmd, capture_output=True, text=True)
    print(name, "ok" if r.returncode == 0 else r.stderr[-2000:])
