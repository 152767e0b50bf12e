"""Mutation check of the oracle pins: apply plausible mistakes to oracle/ldsolver_oracle.py one at a time
and confirm tests/test_oracle_pins.py fails for each (run from the repo root)."""
import subprocess, shutil, sys
src = open('oracle/ldsolver_oracle.py').read()
muts = [
 ("shift=3 - t", "shift=2 - t"),
 ("gamma = 0.5 if system == 0 else 1.0", "gamma = 1.0"),
 ("- alpha * u\n", "+ alpha * u\n"),
 ("@ W[:, ky, kx, :].T", "@ W[:, kx, ky, :].T"),
 ("np.roll(H, shift=(-dy, -dx)", "np.roll(H, shift=(dy, dx)"),
 ("np.sin(kf * y)[:, None]", "np.sin(kf * y)[None, :]"),
 ("kh[n // 2] = 0.0", "pass"),
 ("U2 = self.P(0.75 * u + 0.25 * (U1 + dt * T2))", "U2 = self.P(0.75 * u + 0.25 * (U1 + dt * T1))"),
 ("T1, e = self.T(u)\n", "T1, e = self.T(u)\n        e = None if e is None else e * 0.5\n"),
 ("ux = face_values(u, wIx, -1)", "ux = face_values(u, wDx, -1)"),
 ("(np.roll(Fy, -1, axis=-2) - Fy)", "(np.roll(Fy, 1, axis=-2) - Fy)"),
 ("np.outer(s, s)", "0.0"),
 ("raw[..., 1, :] @ PD.T", "raw[..., 1, :] @ PI.T"),
 ("out = self.P(u / 3.0 + (2.0 / 3.0) * (U2 + dt * T3) + E)", "out = u / 3.0 + (2.0 / 3.0) * (U2 + dt * T3) + E"),
 # R8: e taken from the last stage's net instead of the stage-1 net on u^n (RK3, RK2)
 ("T3, _ = T(U2)\n", "T3, e3 = T(U2)\n            E = e3 if add_e else 0.0\n"),
 ("T2, _ = T(U1)\n            out = self.P(0.5", "T2, e2 = T(U1)\n            E = e2 if add_e else 0.0\n            out = self.P(0.5"),
 # R9: Burgers projected like NS
 ("return project(U, self.h) if self.system == 1 else U", "return project(U, self.h)"),
]
for a, b in muts:
    assert a in src, a
    open('oracle/ldsolver_oracle.py','w').write(src.replace(a, b, 1))
    r = subprocess.run([sys.executable, '-m', 'pytest', 'tests/test_oracle_pins.py', '-x', '-q'], capture_output=True, text=True)
    print(('CAUGHT ' if r.returncode else 'MISSED ') + a[:60])
open('oracle/ldsolver_oracle.py','w').write(src)
