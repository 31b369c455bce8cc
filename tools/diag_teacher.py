"""Diagnostic: teacher-forced per-op errors of one configuration (worst entries).

    RFK_BN_FOLD=<mask> python tools/diag_teacher.py inception_v3 4 299
"""
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from _parity import teacher_forced  # noqa: E402

arch, b, hw = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
res = teacher_forced(arch, b, hw, 1000 if hw >= 224 else 10)
for k in ("fwd", "dgrad", "pgrad"):
    w = sorted(res[k].items(), key=lambda kv: -kv[1])[:4]
    print(os.environ.get("RFK_BN_FOLD", "3"), k, [(n, f"{e:.2e}") for n, e in w])
