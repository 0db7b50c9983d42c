import os, subprocess, sys
for copy in ("memcpy", "nt"):
    for th in ("6", "8", "10", "12"):
        for sl in ("8", "16", "32"):
            env = {**os.environ, "GAPA_PINNED_RING_COPY": copy, "GAPA_PINNED_RING_THREADS": th, "GAPA_PINNED_SLICE_MB": sl}
            subprocess.call([sys.executable, "tools/probe_pageable.py", "child"], env=env)
