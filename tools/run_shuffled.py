"""Runs the GPU test ids in reversed and in shuffled order (finds
test-order-dependent state: caches keyed by buffer addresses, staging
buffers, graph caches)."""
import random
import subprocess
import sys

ids = subprocess.run([sys.executable, "-m", "pytest", "tests", "-m", "gpu", "--collect-only", "-q"],
                     capture_output=True, text=True).stdout.split("\n")
ids = [i for i in ids if "::" in i]
for name, order in (("reversed", ids[::-1]), ("shuffled", random.Random(7).sample(ids, len(ids)))):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *order],
                       capture_output=True, text=True)
    tail = [l for l in r.stdout.split("\n") if l.strip()][-6:]
    print(name, len(order), "\n".join(tail))
