"""Build-time ring-depth sweep (needs a GPU): builds variants with -DSCFA_TUNE_* overrides
in parallel, then times bench.py's cfg2 step with each (SCFA_LIB).  Diagnostics only.

    python scripts/tune.py
"""
import concurrent.futures as cf
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_01160_b200 import build  # noqa: E402

VARIANTS = {
    "base": {},
    "fwd_ns0_3_ns1_2": {"NS0_FWD": 3, "NS1_FWD": 2},
    "dq_ns0_4": {"NS0_DQ": 4},
    "dq_ns1_3": {"NS1_DQ": 3},
    "alt_ns0_4_ns1_4": {"NS0_ALT": 4, "NS1_ALT": 4},
    "alt_ns0_8_ns1_6": {"NS0_ALT": 8, "NS1_ALT": 6},
    "qe_2": {"QE": 2},
    "qe_4": {"QE": 4},
}


def one(name):
    flags = [f"-DSCFA_TUNE_{k}={v}" for k, v in VARIANTS[name].items()]
    out = os.path.join("/tmp/scfa_tune", f"lib_{name}.so")
    try:
        build.build(force=True, out=out, extra=flags)
        return name, out
    except subprocess.CalledProcessError:
        return name, None


with cf.ThreadPoolExecutor(4) as ex:
    libs = dict(ex.map(one, VARIANTS))
for name, lib in libs.items():
    if lib is None:
        print(f"{name:22s} build failed (shared memory budget?)", flush=True)
        continue
    res = []
    for _ in range(2):
        p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "5",
                            "--no-cfg3", "--no-cpu-baseline"], env=dict(os.environ, SCFA_LIB=lib),
                           capture_output=True, text=True, timeout=300)
        try:
            d = json.loads(p.stdout.strip().splitlines()[-1])
            res.append((d["ms_per_step"], d["stages_ms"]))
        except Exception:
            res.append((None, p.stderr[-300:]))
    best = min(r[0] for r in res if r[0]) if any(r[0] for r in res) else None
    st = res[0][1] if isinstance(res[0][1], dict) else {}
    print(f"{name:22s} {best}  fwd {st.get('scfa_attn_fwd')} dq {st.get('scfa_attn_bwd_dq')} "
          f"dkdv {st.get('scfa_attn_bwd_dkdv')}", flush=True)
