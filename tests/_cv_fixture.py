"""Rows of the O12 hand fixture (tests/golden/o12_cv_hand_fixture.json): input construction only."""
import numpy as np


def cv_hand_fixture_rows(g):
    """(X, y, llm_id, prof_id, users_col, n_llm, n_prof) of the 3-LLM x 2-profile x 4-level fixture."""
    X, y, li, pi = [], [], [], []
    for m, name in enumerate(("A", "B", "C")):
        for p in range(2):
            for k, u in enumerate(g["user_levels"]):
                X.append([1.0, float(p), float(u)])
                y.append([g["y1"], float(g["y2"][name][p][k])])
                li.append(m)
                pi.append(p)
    return (np.array(X, np.float32), np.array(y, np.float32), np.array(li, np.int32), np.array(pi, np.int32), 2, 3,
            2)
