"""Run a lab script once per compile-time variant of the library.
  python tools/lab/variant_run.py <script.py> NAME=DEF1,DEF2 ...   (the default build first)
Each variant is built by tools/build.py build_variant into tools/lab/variants/ and
selected through TOPK_LIB; the script's output lines are prefixed with the name."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from tools.build import build_variant, deps  # noqa: E402

script = sys.argv[1]
libs = [("default", None)]
os.makedirs(os.path.join(ROOT, "tools/lab/variants"), exist_ok=True)
for spec in sys.argv[2:]:
    name, _, defs = spec.partition("=")
    out = os.path.join(ROOT, "tools/lab/variants", f"lib_{name}.so")
    if not (os.path.exists(out) and os.path.getmtime(out) > max(os.path.getmtime(f) for f in deps())):
        build_variant(out, [d for d in defs.split(",") if d])  # else prebuilt here (travels with gpurun)
    libs.append((name, out))
for name, lib in libs:
    env = dict(os.environ)
    if lib:
        env["TOPK_LIB"] = lib
    r = subprocess.run([sys.executable, script], env=env, capture_output=True, text=True, timeout=900)
    for line in (r.stdout.strip() or r.stderr[-800:]).splitlines():
        print(f"[{name}] {line}", flush=True)
