"""Mutation check of the C++ oracle's pins: apply plausible mistakes to oracle/cpp/ldsolver_oracle.cpp one
at a time, rebuild, and confirm tests/test_cpp_oracle.py fails for each (run from the repo root)."""
import subprocess
import sys

P = "oracle/cpp/ldsolver_oracle.cpp"
src = open(P).read()
muts = [
    ("wrap(i + kx - 1, N)) * ci]", "wrap(i - kx + 1, N)) * ci]"),                 # conv taps mirrored
    ("f[(size_t)j * N + wrap(i - 3 + t, N)]", "f[(size_t)j * N + wrap(i - 2 + t, N)]"),   # x-face shift
    ("gamma = c.system == 0 ? (R)0.5 : (R)1", "gamma = (R)1"),                     # Burgers flux factor
    ("if (op == 1) p -= s[t] * s[t2] / ss;", ""),                                   # Pi_D loses s s^T
    ("- (R)c.drag * u[(size_t)j * N + i]", "+ (R)c.drag * u[(size_t)j * N + i]"),   # drag sign
    ("const bool null = (mx == 0 || mx == N / 2) && (my == 0 || my == N / 2);",
     "const bool null = mx == 0 && my == 0;"),                                      # Nyquist null modes kept
    ("U2[q] = (R)0.75 * u[q] + (R)0.25 * (Us[q] + dt * Tk[q]);", "U2[q] = (R)0.75 * u[q] + (R)0.25 * (Us[q] + dt * T1[q]);"),
    ("T(u, T1.data(), e.data(), pool);   // e from", "T(u, T1.data(), nullptr, pool);   // e from"),   # TC dropped
    ("if (c.system == 1) project(c, U, pool);", "project(c, U, pool);"),           # Burgers projected (R9)
    ("(fy[(size_t)wrap(j + 1, N) * N + i] - fy[(size_t)j * N + i])", "(fy[(size_t)wrap(j - 1, N) * N + i] - fy[(size_t)j * N + i])"),
    ("const R ux = xface(u, wc + 0);", "const R ux = xface(u, wc + 6);"),           # interp/deriv swap
    ("t += (R)c.force_amp * std::sin((R)c.force_k * y)", "t += (R)c.force_amp * std::cos((R)c.force_k * y)"),
    ("(k + 1) % c.tc_interval == 0", "k % c.tc_interval == 0"),                     # TC gating
]
missed = 0
try:
    for a, b in muts:
        assert a in src, a
        open(P, "w").write(src.replace(a, b, 1))
        r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_cpp_oracle.py", "-x", "-q"],
                           capture_output=True, text=True)
        ok = r.returncode != 0
        missed += not ok
        print(("CAUGHT " if ok else "MISSED ") + a[:70])
finally:
    open(P, "w").write(src)
    subprocess.run([sys.executable, "-c", "from oracle import cpp_oracle as X; X.build(force=True)"])
sys.exit(1 if missed else 0)
