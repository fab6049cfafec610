#!/usr/bin/env python
"""Mutation check of the oracle's pins.

Each mutation is a one-line plausible mistake in oracle/saga_oracle.cpp.  The mutant is compiled
to a temporary library and the CPU pins (tests/test_oracle.py, tests/test_oracle_keys.py) are run
against it through SAGA_ORACLE_LIB.  A mutation is "killed" when at least one pin fails.
Writes profiles/r02_oracle_mutations.md."""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "saga_oracle.cpp")

MUTATIONS = [
    ("tau_max over S (in-flight blocks included)",
     "          for (size_t i = 0; i < cand.size(); ++i) {\n            float s32;",
     "          for (uint32_t b : S) x.tau = std::max(x.tau, Te - tl[b]);\n"
     "          for (size_t i = 0; i < cand.size(); ++i) {\n            float s32;"),
    ("size_max over S (in-flight blocks included)",
     "          for (size_t i = 0; i < cand.size(); ++i) {\n            float s32;",
     "          for (uint32_t b : S) x.smax = std::max(x.smax, owner_state(owner[nd.uniq[b]], e, ev.act).size);\n"
     "          for (size_t i = 0; i < cand.size(); ++i) {\n            float s32;"),
    ("c* with e(c) < e instead of <=", "return ee < ecall[c]; });", "return ee <= ecall[c]; });"),
    ("n_cur = prompt only", "uint64_t ncur = uint64_t(prompt[c]) + outt[c];", "uint64_t ncur = uint64_t(prompt[c]);"),
    ("R and S swapped in eq:eviction", "((cfg.alpha * R) + (cfg.beta * (1.0f - st.P))) + (cfg.gamma * S)",
     "((cfg.alpha * S) + (cfg.beta * (1.0f - st.P))) + (cfg.gamma * R)"),
    ("t_call = t_c instead of the tool start t_end", "st.t_call = t_end(uint32_t(c));", "st.t_call = t[c];"),
    ("beta * P instead of beta * (1 - P)", "(cfg.beta * (1.0f - st.P))", "(cfg.beta * st.P)"),
    ("overlap normalised by n_cur (Eq. 5 form)", "uint64_t den = ncur + nobs;", "uint64_t den = ncur;"),
    ("terminal node ignored in fin", "st.fin = last[c] || term[v];", "st.fin = last[c];"),
    ("pressure sign flipped", "(2 * x.den - x.num)", "(2 * x.den + x.num)"),
    ("TTL_max bound inclusive", "if (!(el < cfg.ttl_max_us)) return false;", "if (!(el <= cfg.ttl_max_us)) return false;"),
    ("occupancy after admission instead of |S| after R1", "make_ctx(cfg, e, Te, int64_t(S.size()), C, ev.act)",
     "make_ctx(cfg, e, Te, int64_t(S.size()) + nnew, C, ev.act)"),
    ("q rounded instead of floored", "float f = std::floor(sc * 1048576.0f);", "float f = std::round(sc * 1048576.0f);"),
    ("unprotected-first order inverted", "keys.push_back({(uint64_t(!pr) << 63)", "keys.push_back({(uint64_t(pr) << 63)"),
    ("shared prefix always P = 1", "st.P = st.act ? 1.0f : 0.0f;", "st.P = 1.0f;"),
    ("argmin ties by highest id", "if (load(x) < load(w)) w = x;", "if (load(x) <= load(w)) w = x;"),
    ("cached TTL bound strict", "(Te - t_end(uint32_t(last_c[s])) <= ttl_of(uint32_t(last_c[s])))",
     "(Te - t_end(uint32_t(last_c[s])) < ttl_of(uint32_t(last_c[s])))"),
    ("steal: newest pending session", "    for (auto& x : q) {\n      if (x.started) continue;",
     "    for (auto it = q.rbegin(); it != q.rend(); ++it) {\n      auto& x = *it;\n      if (x.started) continue;"),
    ("reroute re-prefill counted as compulsory (node first touch)",
     "if (first_call[nd.block[p]] == g.call) ctr[C_COMPULSORY_GLOBAL]++;",
     "if (nd.ftn[p]) ctr[C_COMPULSORY_GLOBAL]++;"),
]


def main():
    src = open(SRC).read()
    rows = []
    tmp = tempfile.mkdtemp(prefix="mut_")
    sel = sys.argv[1:]
    for i, (name, old, new) in enumerate(MUTATIONS):
        if sel and str(i) not in sel:
            continue
        n = src.count(old)
        if n != 1:
            rows.append((name, f"NOT APPLIED (pattern found {n}x)", ""))
            continue
        cpp = os.path.join(tmp, f"m{i}.cpp")
        lib = os.path.join(tmp, f"m{i}.so")
        open(cpp, "w").write(src.replace(old, new))
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", lib, cpp,
                               "-lpthread"])
        env = dict(os.environ, SAGA_ORACLE_LIB=lib)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                            "tests/test_oracle.py", "tests/test_oracle_keys.py", "tests/test_oracle_place.py"],
                           cwd=ROOT, env=env, capture_output=True, text=True)
        failed = [l.split(" ")[1] for l in r.stdout.splitlines() if l.startswith("FAILED")]
        rows.append((name, "killed" if r.returncode else "SURVIVED", failed[0] if failed else ""))
        print(rows[-1], flush=True)
    out = os.path.join(ROOT, "profiles", "r02_oracle_mutations.md")
    with open(out, "w") as f:
        f.write("# Oracle mutation check (scripts/mutate_oracle.py)\n\n")
        f.write("Each row is a one-line mistake applied to oracle/saga_oracle.cpp; the not-gpu oracle pins are run "
                "against the mutant.  `killed` = at least one pin fails (first failure shown).\n\n")
        f.write("| # | Mutation | Result | First failing pin |\n|---|---|---|---|\n")
        for i, (name, res, t) in enumerate(rows):
            f.write(f"| {i} | {name} | {res} | `{t}` |\n")
    print(out)


if __name__ == "__main__":
    main()
