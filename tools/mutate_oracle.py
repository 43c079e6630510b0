"""Mutation check of the oracle's pins.

Copies the repo to a temp dir, applies one source mutation at a time to
oracle/distir_oracle.cpp, rebuilds the oracle there and runs the CPU tier
(`-m "not gpu"`, the oracle pins only).  Every mutation must turn at least one
test red.  Usage: python tools/mutate_oracle.py [> profiles/r02_oracle_mutations.txt]
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "oracle/distir_oracle.cpp"

# (name, old, new): each `old` must occur exactly once in the oracle source.
MUTATIONS = [
    ("M1 AllGather bandwidth term without (g-1)/g",
     "    return ((double)(g - 1)) * a +\n           (((double)(g - 1)) / ((double)g)) * (((double)op.work) / bw);",
     "    return ((double)(g - 1)) * a +\n           (((double)op.work) / bw);"),
    ("M2 link class always intra-node",
     "    if (d / t.node_size != devs[0] / t.node_size) return false;",
     "    if (false) return false;"),
    ("M3 AllReduce alpha steps (g-1) instead of 2(g-1)",
     "    return ((double)(2 * (g - 1))) * a +",
     "    return ((double)(g - 1)) * a +"),
    ("M3b AllReduce alpha steps fixed at 2",
     "    return ((double)(2 * (g - 1))) * a +",
     "    return ((double)2) * a +"),
    ("M4 GPT-2 block parameters never freed",
     "for (int q = 0; q < NPB; q++) bp[(r * L + l) * NPB + q] = pr.new_val(r, pbytes[q], true);",
     "for (int q = 0; q < NPB; q++) bp[(r * L + l) * NPB + q] = pr.new_val(r, pbytes[q], true, true);"),
    ("M5 GPT-2 residual outputs never freed",
     "          x3[r] = pr.new_val(r, n * d * e);",
     "          x3[r] = pr.new_val(r, n * d * e, false, true);"),
    ("M6 AllReduce bandwidth factor 1 instead of 2(g-1)/g",
     "           (((double)(2 * (g - 1))) / ((double)g)) * (((double)op.work) / bw);",
     "           (((double)op.work) / bw);"),
    ("M7 GPT-2 attention scores freed early (qkv dead after scores)",
     "          emit(COMPUTE, {r}, {pb[r], qkv[r]}, {ctx[r]}, 2 * m * S * S * dT, true);",
     "          emit(COMPUTE, {r}, {pb[r]}, {ctx[r]}, 2 * m * S * S * dT, true);"),
    ("M8 Send uses intra constants always",
     "  const bool in_node = intra(t, op.devs);",
     "  const bool in_node = op.cls == SEND ? true : intra(t, op.devs);"),
    ("M9 GPT-2 logits shard kept after AllGather",
     "            int lg = pr.new_val(r, n * VT * e, false, T == 1);",
     "            int lg = pr.new_val(r, n * VT * e, false, true);"),
]

TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_pins_comm_memory.py",
         "tests/test_oracle_1f1b.py", "tests/test_oracle_f4.py",
         "tests/test_oracle_regression.py"]


def run(tmp):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu",
                        "-rf", "-p", "no:cacheprovider"] + TESTS,
                       cwd=tmp, capture_output=True, text=True)
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    failed = [l.split()[1] for l in lines if l.startswith("FAILED ")]
    return r.returncode, failed + lines[-1:]


def main():
    src = open(os.path.join(ROOT, SRC)).read()
    tmp = tempfile.mkdtemp(prefix="mut_")
    shutil.copytree(ROOT, tmp, dirs_exist_ok=True,
                    ignore=shutil.ignore_patterns(".git", "gpurun_out", "liboracle.so", "__pycache__"))
    rc, tail = run(tmp)
    print("baseline (unmutated): exit %d  %s" % (rc, tail[-1] if tail else ""))
    assert rc == 0, "unmutated oracle must pass"
    survivors = 0
    for name, old, new in MUTATIONS:
        assert src.count(old) == 1, "mutation anchor not unique: " + name
        open(os.path.join(tmp, SRC), "w").write(src.replace(old, new))
        so = os.path.join(tmp, "oracle", "liboracle.so")
        if os.path.exists(so):
            os.remove(so)
        rc, tail = run(tmp)
        killed = rc != 0
        survivors += not killed
        print("%-62s %s  %s" % (name, "KILLED  by" if killed else "SURVIVED", tail[0][:120]))
    open(os.path.join(tmp, SRC), "w").write(src)
    shutil.rmtree(tmp, ignore_errors=True)
    print("survivors: %d of %d" % (survivors, len(MUTATIONS)))
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
