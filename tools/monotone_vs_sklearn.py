"""Why the synthetic C2 cross-validation scores low (bench cv_c2: S = 3 %): the monotone constraint
 implemented as XGBoost does — users splits need wL <= wR, children bounded by the
midpoint (wL + wR) / 2, leaf weights clamped to their bounds — stalls on targets whose residuals
are not monotone in every subtree and can drive predictions negative.  scikit-learn's
HistGradientBoostingRegressor(monotonic_cst=...) uses the same midpoint rule and shows the same
behaviour on a toy target y = (a + 1) u / 2 + 3 that is monotone in u.

    python tools/monotone_vs_sklearn.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from sklearn.ensemble import HistGradientBoostingRegressor  # noqa: E402

import oracle  # noqa: E402

rng = np.random.default_rng(0)
n = 2000
a = rng.integers(0, 10, n).astype(np.float32)
u = rng.choice([1, 2, 4, 8, 16, 32, 64, 128], n).astype(np.float32)
y = (a + 1) * u * 0.5 + 3
X = np.stack([a, u], 1).astype(np.float32)
print("%-10s %-5s %6s %10s %10s %10s" % ("model", "mono", "trees", "med.rel", "max.abs", "min.pred"))
for mono in (0, 1):
    for T in (10, 50, 200):
        _, tp = oracle.fit(X, np.stack([y, y], 1), oracle.hparams(n_trees=T, max_depth=4, use_eq4_weights=0,
                                                                  monotone_users=mono), 1, return_train_pred=True)
        p = tp[:, 0]
        print("%-10s %-5d %6d %10.4f %10.2f %10.2f" % ("oracle", mono, T, np.median(np.abs(p / y - 1)),
                                                       np.abs(p - y).max(), p.min()))
        m = HistGradientBoostingRegressor(max_iter=T, max_depth=4, learning_rate=0.3, l2_regularization=1.0,
                                          min_samples_leaf=1, monotonic_cst=[0, mono], early_stopping=False).fit(X, y)
        p = m.predict(X)
        print("%-10s %-5d %6d %10.4f %10.2f %10.2f" % ("sklearn", mono, T, np.median(np.abs(p / y - 1)),
                                                       np.abs(p - y).max(), p.min()))
