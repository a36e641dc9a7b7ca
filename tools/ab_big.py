import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for lib in sys.argv[1:]:
    env = dict(os.environ, KMB_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "big_threads.py")], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), (r.stdout.strip().splitlines() or [r.stderr[-300:]])[-1], flush=True)
