# Per-stage device times of one solve with the S-digit cache off and on
# (DSB_TRACE stage marks): python tools/sdig_probe.py n k p [euclid|f32|ham] [q]
import os
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def run(args, cache):
    env = dict(os.environ, DSB_TRACE="1", DSB_SDIG=str(cache))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_1803_02272_b200 as ds\n"
        "n, k, p, kind, q = %d, %d, %d, %r, %d\n"
        "ds.set_device(0); ds.set_product_path(2)\n"
        "if kind == 'ham':\n"
        "    D = ds.matrix_hamming(ds.synth_reads(n, 400, 50, 0.05, 3))\n"
        "else:\n"
        "    D = ds.matrix_euclidean(ds.synth_points(3, n, 3), store_f32=(kind == 'f32'))\n"
        "g = ds.gram(D)\n"
        "for _ in range(2):\n"
        "    ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=1)\n"
        "print('sdig', ds.stats_get().last_product_sdig, file=sys.stderr)\n"
    ) % (str(ROOT), *args)
    err = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                         text=True).stderr
    lines = err.splitlines()
    # the last solve's stage marks
    start = max(i for i, ln in enumerate(lines) if "host enqueue done" in ln)
    marks = [ln for ln in lines[start:] if re.match(r"\[trace\] \S+\s+[\d.]+ us$", ln)]
    prod = [float(ln.split()[-2]) for ln in marks if ln.split()[1] == "product"]
    tot = sum(float(ln.split()[-2]) for ln in marks)
    sd = [ln for ln in lines if ln.startswith("sdig")]
    return prod, tot, sd[-1] if sd else "?"


if __name__ == "__main__":
    n, k, p = (int(x) for x in sys.argv[1:4])
    kind = sys.argv[4] if len(sys.argv) > 4 else "euclid"
    q = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    for cache in (0, 2):
        prod, tot, sd = run((n, k, p, kind, q), cache)
        print(f"n={n} w={k + p} {kind} cache={cache} ({sd}): product passes (us) "
              + " ".join(f"{x:.0f}" for x in prod) + f" | solve {tot:.0f} us")
