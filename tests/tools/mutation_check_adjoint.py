"""Mutation check of the adjoint oracle's pins (oracle/adjoint_oracle.py vs tests/test_adjoint_oracle.py)."""
import subprocess
import sys

P = "oracle/adjoint_oracle.py"
src = open(P).read()
muts = [
    ("np.roll(G, shift=(dy, dx), axis=(1, 2))", "np.roll(G, shift=(-dy, -dx), axis=(1, 2))"),
    (" + x * np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)", ""),
    ("Fxbar = -(np.roll(Tbar[:, ci], 1, axis=-1) - Tbar[:, ci]) / h", "Fxbar = -(np.roll(Tbar[:, ci], -1, axis=-1) - Tbar[:, ci]) / h"),
    ("uxbar += gamma * cx * Fxbar", "uxbar += cx * Fxbar"),
    ("dcybar = -nu * Fybar / h", "dcybar = -nu * Fybar"),
    ("r[..., 1, :] = wbar[..., 1, :] @ PD", "r[..., 1, :] = wbar[..., 1, :] @ PI"),
    ("def _Pt(self, X):   # P is an orthogonal projector (G_c = -D_c^T): self-adjoint\n        return self.P(X)",
     "def _Pt(self, X):   # P is an orthogonal projector (G_c = -D_c^T): self-adjoint\n        return X"),
    ("ebar if s == 0 else None", "ebar if s == len(coef) - 1 else None"),
    ("Ubar -= alpha * Tbar", "Ubar += alpha * Tbar"),
    ("K3b = K3b + dt * p4", "K3b = K3b + 0.5 * dt * p4"),
    ("out += np.roll(w_axis_op[..., t] * gbar, shift=-(3 - t), axis=axis)", "out += w_axis_op[..., t] * np.roll(gbar, shift=-(3 - t), axis=axis)"),
]
missed = 0
try:
    for a, b in muts:
        assert a in src, a
        open(P, "w").write(src.replace(a, b, 1))
        r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_adjoint_oracle.py", "-x", "-q"],
                           capture_output=True, text=True)
        ok = r.returncode != 0
        missed += not ok
        print(("CAUGHT " if ok else "MISSED ") + a[:70].replace("\n", " "))
finally:
    open(P, "w").write(src)
sys.exit(1 if missed else 0)
