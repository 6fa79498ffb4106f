"""Mutation check of the GPU parity tests: one-line mutants of the CUDA sources, each built into
variants/mut_<k>.so; `--run` (on a B200) loads each through QVTS_LIB and runs a fast subset of the
`-m gpu` parity tests, which must fail.  `python tests/cuda_mutations.py --build` here (nvcc
cross-compiles), then `python tests/cuda_mutations.py --run` on the GPU box.  Prints JSON."""
import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))   # repo root (this file: tests/)
CSRC = os.path.join(ROOT, "paper_1810_00204_b200", "csrc")
OUT = os.path.join(ROOT, "variants")

MUTANTS = [
    ("S4: correct without the 1/P(z) normaliser", "plan.cu",
     "s_w[sg][u] = pz > 1e-30 ? (float)(a.O64[sg * 16 + z] / pz) : 0.f;",
     "s_w[sg][u] = pz > 1e-30 ? (float)(a.O64[sg * 16 + z]) : 0.f;"),
    ("S3: Philox key halves swapped", "plan.cu", "make_uint2(a.seed, ep));", "make_uint2(ep, a.seed));"),
    ("S6: gamma dropped in the backup", "plan.cu", "qv = R[q] + gamma * acc;", "qv = R[q] + acc;"),
    ("S1: lateral ring neighbour off by one", "stencil.cuh", "return ring_at((ring_pos(k) + 7) % 8);",
     "return ring_at((ring_pos(k) + 6) % 8);"),
    ("S1/S2 (k_hist): diagonal blocked mass not kept at y", "plan.cu", "                h += b0;\n", "\n"),
    ("NEXT-1: gamma dropped in the FIB sweep", "model.cu", "out = R64[(size_t)j * HW + x] + gamma * s;",
     "out = R64[(size_t)j * HW + x] + s;"),
    ("S7: gamma dropped in value iteration", "model.cu", "    return R64[(size_t)j * HW + x] + gamma * s;\n}",
     "    return R64[(size_t)j * HW + x] + s;\n}"),
    ("NEXT-2: PBVI alpha* by the first instead of the best vector", "pbvi.cu", "if (k == 0 || pb_beats(v, bz)) { bz = v; bk = k; }",
     "if (k == 0) { bz = v; bk = k; }"),
    ("S2: R(b,a) identity with p_stay instead of p_stay - 1", "plan.cu", "R = (a.p_stay - 1.0) * mass - Rp + gsum;",
     "R = a.p_stay * mass - Rp + gsum;"),
    ("S4 (staged k_correct): left neighbour read from the cell itself", "plan.cu", "nbh[dr][0] = row[-1];",
     "nbh[dr][0] = row[0];"),
    ("S2 (k_reduce band sum): second element of a pair summed from the first", "plan.cu",
     "if (bd + u < a.nb) { acc0 += x[u].x; acc1 += x[u].y; }", "if (bd + u < a.nb) { acc0 += x[u].x; acc1 += x[u].x; }"),
    ("S5: leaf offset qbar not added back", "plan.cu", "const double Vz = a.qbar + best / Pz;",
     "const double Vz = best / Pz;"),
    ("best-first Alg. 7: heuristic child by H instead of U", "bestfirst.cu", "if (U[j] > U[bq]) bq = j;",
     "if (H[j] > H[bq]) bq = j;"),
    # round 2 kernels
    ("S5 (k_leaf): every b product with the first Q' column", "leaf.cu",
     "for (int j = 0; j < NA; ++j) F[0][j] = ffma2s(b0, q[j], F[0][j]);",
     "for (int j = 0; j < NA; ++j) F[0][j] = ffma2s(b0, q[0], F[0][j]);"),
    ("S1 (k_leaf): diagonal blocked mass not kept at y", "leaf.cu", "hd[i] = fadd2(b0, hd[i]);", "hd[i] = hd[i];"),
    ("S2 (k_leaf TMEM fold): class masses of the two parents swapped", "leaf.cu",
     "d += (double)((i & 1) ? S[f].y : S[f].x);", "d += (double)((i & 1) ? S[f].x : S[f].y);"),
    ("S2 (k_reduce): sensor butterfly with acc and 1 - acc swapped", "plan.cu",
     "Pz = fma(ka, Pz, kb * __shfl_xor_sync(0xffffffffu, Pz, bt));",
     "Pz = fma(kb, Pz, ka * __shfl_xor_sync(0xffffffffu, Pz, bt));"),
    ("S5 (k_reduce): leaf numerator butterfly with acc and 1 - acc swapped", "plan.cu",
     "Sv[j2] = fma(ka, Sv[j2], kb * __shfl_xor_sync(0xffffffffu, Sv[j2], bt));",
     "Sv[j2] = fma(kb, Sv[j2], ka * __shfl_xor_sync(0xffffffffu, Sv[j2], bt));"),
    ("K9 (k_bu_cluster): a lateral's blocked mass not kept at y", "plan.cu",
     "if ((t >> nbit(k1)) & 1) c += a.p_lat;", "if ((t >> nbit(k1)) & 1) c += 0.f;"),
    ("K9 (k_bu_cluster): the normaliser of rank 0's rows only", "plan.cu", "P += s_parts[rr];", "P += s_parts[0];"),
    ("NEXT-3 (k_ancestral_x): the in-chunk scan starts one chunk late", "plan.cu", "double acc = cpre[lo];",
     "double acc = cpre[lo + 1];"),
]
SUBSET = ("test_tables_and_value_iteration or test_belief_update or test_plan_C1_full_tree or "
          "test_plan_ragged_depth3 or test_plan_C3_full or test_best_first_against_oracle or "
          "test_pbvi_against_oracle or test_plan_ancestral_sampler")   # C3 (W = 128): staged k_correct,
# k_leaf with several bands; test_belief_update*: the cluster kernel (C3, cluster shapes)


def build():
    os.makedirs(OUT, exist_ok=True)
    res = []
    for k, (name, fname, old, new) in enumerate(MUTANTS):
        with tempfile.TemporaryDirectory() as tmp:
            d = os.path.join(tmp, "pkg", "csrc")          # csrc/../../include -> tmp/include
            shutil.copytree(CSRC, d, ignore=shutil.ignore_patterns("*.o", "*.log"))
            shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
            path = os.path.join(d, fname)
            src = open(path).read()
            if src.count(old) != 1:
                res.append({"mutant": name, "status": f"pattern count {src.count(old)}"})
                continue
            open(path, "w").write(src.replace(old, new))
            lib = os.path.join(OUT, f"mut_{k}.so")
            r = subprocess.run(["make", "-s", "-j4", "-C", d, f"LIB={lib}"], capture_output=True, text=True)
            res.append({"mutant": name, "lib": os.path.basename(lib), "built": r.returncode == 0,
                        "err": r.stderr[-300:] if r.returncode else ""})
        print(json.dumps(res[-1]), flush=True)
    json.dump(res, open(os.path.join(OUT, "mutants.json"), "w"))


def run():
    res = json.load(open(os.path.join(OUT, "mutants.json")))
    caught = 0
    for r in res:
        if not r.get("built"):
            continue
        env = dict(os.environ, QVTS_LIB=os.path.join(OUT, r["lib"]))
        p = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                            "-k", SUBSET, os.path.join(ROOT, "tests", "test_gpu_parity.py")], cwd=ROOT, env=env,
                           capture_output=True, text=True, timeout=900)
        r["caught"] = p.returncode != 0
        r["first_failing"] = [l.split("::")[-1][:80] for l in p.stdout.splitlines() if l.startswith("FAILED")][:1]
        caught += r["caught"]
        print(json.dumps(r), flush=True)
    print(json.dumps({"caught": caught, "total": len(res), "mutants": res}))


if __name__ == "__main__":
    build() if "--build" in sys.argv else run()
