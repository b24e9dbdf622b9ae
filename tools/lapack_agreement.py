"""Writes oracle/lapack.py's canonical-vs-LAPACK comparison for the named configs, one JSON
object per line (profiles/r02_lapack_agreement.jsonl)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.lapack import compare  # noqa: E402

if __name__ == "__main__":
    for name in sys.argv[1:] or ["C1", "C2", "C5/4", "C4i", "C4iii"]:
        print(json.dumps(compare(name)), flush=True)
