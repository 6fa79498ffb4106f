"""Mutation check of the oracle's pins (task rule 3: a plausible mistake anywhere -- a dropped term,
a wrong sign or index, a transposed operand -- must fail a `-m "not gpu"` pin).  Each mutant is
a one-line edit of oracle/qvts_oracle.c built into /tmp; tests/test_oracle_pins.py runs against it
through QVTS_ORACLE_LIB and must fail.  Prints one JSON object (caught / total, per mutant)."""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))   # repo root (this file: tests/)
SRC = open(os.path.join(ROOT, "oracle", "qvts_oracle.c")).read()

MUTANTS = [
    ("uniform: drop the +0.5 centring", "((double)(w >> 8) + 0.5)", "((double)(w >> 8) + 0.0)"),
    ("inverse CDF: <= instead of <", "if (t < C[k]) { res = k; break; }", "if (t <= C[k]) { res = k; break; }"),
    ("predict: transposed T (gather by x)", "bbar[m->t_y[e]] += m->t_p[e] * b[x];", "bbar[x] += m->t_p[e] * b[m->t_y[e]];"),
    ("marginal: O index transposed", "s += m->O[y * m->nz + z] * bbar[y];", "s += m->O[z * m->nz + y % m->nz] * bbar[y];"),
    ("belief update: drop the normaliser", "out[y] = m->O[y * m->nz + z] * bbar[y] / pz;", "out[y] = m->O[y * m->nz + z] * bbar[y];"),
    ("sensor: accuracy swapped", "((m->sig[x] >> k) & 1)) ? acc : (1.0 - acc);", "((m->sig[x] >> k) & 1)) ? (1.0 - acc) : acc;"),
    ("laterals: wrong ring neighbour", "w[RING[(i + 7) % 8]] += p_lat;", "w[RING[(i + 6) % 8]] += p_lat;"),
    ("clamp: blocked mass dropped", "if (o) y = x;                       /* clamp */", "if (o) continue;"),
    ("reward: collision worth -1", "double r = o ? -2.0 : (y == goal ? 0.0 : -1.0);", "double r = o ? -1.0 : (y == goal ? 0.0 : -1.0);"),
    ("reward: stay off goal worth -1", "else if (m->action_id[a] == 4 && x != goal) v = -2.0;", "else if (m->action_id[a] == 4 && x != goal) v = -1.0;"),
    ("VI: gamma dropped", "return m->R[x * m->na + a] + m->gamma * s;", "return m->R[x * m->na + a] + s;"),
    ("FIB: sum instead of max over a'", "if (d > best) best = d;", "best = (best == -INFINITY ? 0.0 : best) + d;"),
    ("FIB: start at R_min", "if (!(m->is_grid && m->occ[i / na]) && m->R[i] > rmax) rmax = m->R[i];",
     "if (!(m->is_grid && m->occ[i / na]) && m->R[i] < rmax) rmax = m->R[i];"),
    ("plan backup: gamma dropped", "double Qv = R + m->gamma * acc;", "double Qv = R + acc;"),
    ("plan: weights P instead of f/n", "double w = (cfg->mode == OR_MODE_FREQ) ? (double)cnt[z] / (double)n : P[z];",
     "double w = P[z];"),
    ("best-first Alg. 6: gamma dropped in U_Q", "*UQ = R + gamma * su;", "*UQ = R + su;"),
    ("best-first Alg. 6: heuristic without weight", "double h = gamma * w[c] * H[c];", "double h = gamma * H[c];"),
    ("best-first Alg. 7: H of the larger-H child", "if (UQ[a] > UQ[bq]) bq = a;", "if (HQ[a] > HQ[bq]) bq = a;"),
    ("PBVI: backup with a wrong action index", "out[x] = m->R[x * na + best_a] + m->gamma * acc;",
     "out[x] = m->R[x * na + (best_a + 1) % na] + m->gamma * acc;"),
    ("PBVI: blind start at R_max", "if (!(m->is_grid && m->occ[i / na]) && m->R[i] < rmin) rmin = m->R[i];",
     "if (!(m->is_grid && m->occ[i / na]) && m->R[i] > rmin) rmin = m->R[i];"),
    ("advance: paths not re-based", "        v->path >>= 8;\n", "\n"),
    ("PBVI expansion: nearest candidate", "if (pbvi_beats(dmin, best_d)) { best_d = dmin; best_a = a; }",
     "if (dmin > 0.0 && (best_a < 0 || dmin < best_d)) { best_d = dmin; best_a = a; }"),
    ("PBVI expansion: first candidate off the set", "if (pbvi_beats(dmin, best_d)) { best_d = dmin; best_a = a; }",
     "if (best_a < 0 && dmin > 0.0) { best_d = dmin; best_a = a; }"),
    ("replay: any category accepted", "borders_near_boundary(P, nz, u, zr))", "1)"),
    ("ancestral replay: any state accepted", "&& borders_near_boundary(b, m->nx, or_uniform(w[1]), xr))", ")"),
]

cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
out, caught = [], 0
with tempfile.TemporaryDirectory() as tmp:
    for name, old, new in MUTANTS:
        if SRC.count(old) != 1:
            out.append({"mutant": name, "status": "pattern not unique/absent", "count": SRC.count(old)})
            continue
        src = os.path.join(tmp, "m.c")
        open(src, "w").write(SRC.replace(old, new))
        so = os.path.join(tmp, f"lib_{len(out)}.so")
        b = subprocess.run([cc, "-O2", "-std=c11", "-fPIC", "-ffp-contract=off", "-shared", "-fopenmp",
                            "-I", os.path.join(ROOT, "oracle"), "-o", so, src, "-lm"], capture_output=True)
        if b.returncode:
            out.append({"mutant": name, "status": "build failed"})
            continue
        env = dict(os.environ, QVTS_ORACLE_LIB=so)
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                            os.path.join(ROOT, "tests", "test_oracle_pins.py")], cwd=ROOT, env=env,
                           capture_output=True, text=True, timeout=900)
        ok = r.returncode != 0
        caught += ok
        failed = [l.split("::")[-1].split(" ")[0] for l in r.stdout.splitlines() if l.startswith("FAILED")]
        out.append({"mutant": name, "caught": ok, "first_failing_pin": failed[:1]})
        print(json.dumps(out[-1]), flush=True)
print(json.dumps({"caught": caught, "total": len(MUTANTS), "mutants": out}))
