"""Build tuning variants of libfdtdrom.so (variants/<name>.so, selected at run time with FDTD_LIB)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1609_07114_b200 import build  # noqa: E402


def main(specs):
    os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
    jobs = []
    for spec in specs:  # name=DEF1,DEF2
        name, _, defs = spec.partition("=")
        jobs.append((name, [d for d in defs.split(",") if d]))
    with ThreadPoolExecutor(4) as ex:
        outs = list(ex.map(lambda j: build.build(force=True, out=os.path.join(ROOT, "variants", j[0] + ".so"),
                                                 defines=j[1]), jobs))
    for (name, _), out in zip(jobs, outs):
        print(name, out)


if __name__ == "__main__":
    main(sys.argv[1:])
