"""Build tuning variants of libdbp.so into build_var/<name>.so (-D defines), for A/B timing on
the GPU with DBP_LIB=build_var/<name>.so.  usage: python scripts/build_variants.py name:DEF=V,DEF=V ..."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_04458_b200 import build  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(spec):
    name, _, defs = spec.partition(":")
    out = os.path.join(ROOT, "build_var", name + ".so")
    build.build(force=True, out=out, defines=[d for d in defs.split(",") if d])
    return out


with ThreadPoolExecutor(max_workers=2) as ex:
    for o in ex.map(one, sys.argv[1:]):
        print(o)
