"""sha256 over the kernel sources (paper_1911_09548_b200/csrc/*): tags ncu captures with the code
that produced them (bench.py compares it with the current sources)."""
import glob
import hashlib
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def srchash():
    h = hashlib.sha256()
    for p in sorted(glob.glob(os.path.join(ROOT, "paper_1911_09548_b200", "csrc", "*"))):
        h.update(os.path.basename(p).encode())
        h.update(open(p, "rb").read())
    return h.hexdigest()[:16]


if __name__ == "__main__":
    print(srchash())
