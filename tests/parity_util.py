"""Helpers shared by the GPU parity tests: the R13/R14 definitions live in oracle/tolerance.py
(one definition for tests, smoke() and bench.py's equivalence gate)."""
from oracle.tolerance import (SVM_FLOOR, SVM_RTOL, check_svm, clear_rows,  # noqa: F401
                              labels_agree_away_from_ties, svm_tolerance_ok, top_score_ok)
