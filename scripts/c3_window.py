"""Time the c3 KSE-Parareal window alone (bench.py's parareal field); env knobs
PW_SWEEP_OVERLAP / PW_COOP_CAP are read by the library at context creation."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    out = bench.parareal_c3(0)
    out["env"] = {k: os.environ.get(k) for k in ("PW_SWEEP_OVERLAP", "PW_COOP_CAP")}
    print(json.dumps(out))
