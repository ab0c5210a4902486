"""Time one KSE-Parareal window (bench.py's parareal field) of config c3 (default) or c4:

    python scripts/c3_window.py [c3|c4] [--cold]

Env knobs PW_SWEEP_OVERLAP / PW_COOP_CAP are read by the library at context creation."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out = bench.parareal_window(args[0] if args else "c3", warm="--cold" not in sys.argv)
    out["env"] = {k: os.environ.get(k) for k in ("PW_SWEEP_OVERLAP", "PW_COOP_CAP")}
    print(json.dumps(out))
