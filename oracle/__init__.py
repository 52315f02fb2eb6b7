"""CPU oracle package — TEST INFRASTRUCTURE ONLY.

`oracle.ixo` wraps the plain-C restatement (oracle/ixo.c) and `oracle.ref`
wraps the unmodified reference library compiled in place (oracle/_ref).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs may import this package; the product (paper_2510_17505_b200) never does.
"""
import os
import subprocess

ORACLE_DIR = os.path.dirname(os.path.abspath(__file__))


def build(quiet=True):
    """Builds libixo.so and (when /root/reference is present) oracle/_ref."""
    out = subprocess.run(["make", "-C", ORACLE_DIR, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)
