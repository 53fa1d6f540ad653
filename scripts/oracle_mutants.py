"""Mutation check of the oracle's pins ("each of these mutations passes all pins").

Builds mutated copies of oracle/gpcg_oracle.c under /tmp -- each a plausible mistake in one
rule of Algorithm GPCG -- and runs the -m "not gpu" oracle pins against each (ORACLE_LIB
points oracle.py at the mutant).  A mutant must FAIL at least one pin; the script prints a
table and exits non-zero if any mutant survives.  Never touches the in-tree build.

    python scripts/oracle_mutants.py [-k MUTANT]

(Applying pgstop2 from j >= 1 instead of j >= 2 is an equivalent mutant, not listed: before
the first step the decrease history is empty, max = 0, and every accepted step decreases q.)
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "gpcg_oracle.c")

# name -> (passage, original text, mutated text)
MUTANTS = {
    "pgstop1_removed": ("Eq. pgstop1 P:381-383", "int reason = same ? 1 :", "int reason = 0 ? 1 :"),
    "pgstop1_always": ("Eq. pgstop1 P:381-383", "int reason = same ? 1 :", "int reason = 1 ? 1 :"),
    "pgstop2_uses_eta2": ("Eq. pgstop2 P:386-388", "(j >= 2 && dec <= prm->eta1 * maxdec)",
                          "(j >= 2 && dec <= prm->eta2 * maxdec)"),
    "pgstop2_removed": ("Eq. pgstop2 P:386-388", "(j >= 2 && dec <= prm->eta1 * maxdec)", "(0)"),
    "eta2_never_reduced": ("Eq. cgstop3 P:485-493", "eta2 = eta2 * prm->eta2_shrink;", "eta2 = eta2 * 1.0;"),
    "cgstop3_inverted": ("Eq. cgstop3 P:487-488", "if (nonbinding != 0) break;", "if (nonbinding == 0) break;"),
    "cgstop3_never_refines": ("Eq. cgstop3 P:487-488", "if (nonbinding != 0) break;", "break;"),
    "cgstop1_uses_eta1": ("Eq. cgstop1 P:450-454", "int stop = (it >= 2 && dec <= eta2 * maxdec)",
                          "int stop = (it >= 2 && dec <= 0.1 * maxdec)"),
    "gp_direction_sign": ("Eq. next-y P:341", "for (int64_t i = 0; i < n; i++) w[i] = -g[i];",
                          "for (int64_t i = 0; i < n; i++) w[i] = g[i];"),
    "sufficient_decrease_mu0": ("Eq. gplsstop P:347", "if (dq <= mu * gs) {", "if (dq <= 0.0 * gs) {"),
}

PINS = ["tests/test_oracle_control.py", "tests/test_oracle_pins.py"]


def build(src_text, out):
    with tempfile.NamedTemporaryFile("w", suffix=".c", delete=False) as f:
        f.write(src_text)
        c = f.name
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c99", "-D_POSIX_C_SOURCE=199309L",
                           "-fPIC", "-shared", "-w", "-o", out, c, "-lm"])
    os.unlink(c)


def main():
    only = sys.argv[sys.argv.index("-k") + 1] if "-k" in sys.argv else None
    base = open(SRC).read()
    survivors = []
    for name, (cite, old, new) in MUTANTS.items():
        if only and name != only:
            continue
        assert base.count(old) == 1, (name, base.count(old))
        lib = os.path.join(tempfile.gettempdir(), f"liboracle_{name}.so")
        build(base.replace(old, new), lib)
        env = dict(os.environ, ORACLE_LIB=lib)
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                            "--timeout=900"] + PINS, cwd=ROOT, env=env, capture_output=True, text=True)
        killed = r.returncode != 0
        first = next((ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")), "")
        print(f"{name:26s} {cite:26s} {'killed' if killed else 'SURVIVED'}  {first[:110]}", flush=True)
        if not killed:
            survivors.append(name)
    sys.exit(1 if survivors else 0)


if __name__ == "__main__":
    main()
