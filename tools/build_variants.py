"""Side builds of experimental kernel variants (A/B on the GPU box).

    python tools/build_variants.py NAME:DEF=V[,DEF=V...] ...

builds paper_1908_04081_b200/_lib/libsscg_NAME.so with those -D defines
(a bare value V means SSCG_ROWDOT=V, the original form)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_04081_b200 import build
for v in sys.argv[1:]:
    if ":" in v:
        name, defs = v.split(":", 1)
        defines = tuple(d for d in defs.split(",") if d)
    else:
        name, defines = f"v{v}", (f"SSCG_ROWDOT={v}",)
    print(build.build(out=os.path.join(build.OUT_DIR, f"libsscg_{name}.so"), defines=defines))
