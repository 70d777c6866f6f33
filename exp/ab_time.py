"""A/B of two library builds on one box: python exp/ab_time.py <config> <kernel> <libA> <libB> [reps]
(each timing in its own process through ENS_LIB_PATH, alternating A, B)."""
import os, subprocess, sys
cfg, kernel, la, lb = sys.argv[1:5]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
here = os.path.dirname(os.path.abspath(__file__))
for r in range(reps):
    for tag, lib in (("A", la), ("B", lb)):
        env = dict(os.environ, ENS_LIB_PATH=os.path.abspath(lib))
        K = "500" if cfg in ("c2", "c3") else "100"
        out = subprocess.run([sys.executable, os.path.join(here, "f3_time.py"), cfg, "auto", K, kernel],
                             capture_output=True, text=True, env=env).stdout.strip().splitlines()
        print(tag, out[-1] if out else "no output", flush=True)
