"""Build A/B variants of libtsqr.so into build_ab/<name>.so (developer tool).
usage: python tools/ab_build.py name:-DFLAG[,-DFLAG2] ..."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0808_2664_b200 import _build  # noqa: E402

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.makedirs(os.path.join(root, os.environ.get("AB_DIR", "build_ab")), exist_ok=True)


def one(spec):
    name, _, flags = spec.partition(":")
    out = os.path.join(root, os.environ.get("AB_DIR", "build_ab"), name + ".so")
    _build.build_variant(out, [f for f in flags.split(",") if f], force=True)
    return out


for spec in sys.argv[1:]:        # sequential: build_variant swaps module globals
    print("built", one(spec), flush=True)
