"""Side builds of experimental kernel variants (A/B on the GPU box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_04081_b200 import build
for v in sys.argv[1:]:
    print(build.build(out=os.path.join(build.OUT_DIR, f"libsscg_v{v}.so"), defines=(f"SSCG_ROWDOT={v}",)))
