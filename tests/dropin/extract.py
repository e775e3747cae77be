"""TEST INFRASTRUCTURE ONLY. Extracts, at build time, the reference's own CALLERS of its training API —
run_train + CommonFlags (proj/tools/main.cpp:26-38, :56-101) and the train_run / grad_run test cases of
proj/tests/test_gcn.cpp:213-348 with their dataset helpers (:11-64) — into tests/dropin/_build/*.inc
(git-ignored, never committed), so tests/dropin/dropin_main.cpp compiles them UNCHANGED against
include/mggcn/rowgcn.hpp. The only rewrite is S = double -> float in the test cases (the B200 step trains
in fp32; rowgcn<double> is rejected at compile time by design).

    python tests/dropin/extract.py [/root/reference]      -> exit 3 when the reference is absent
"""
import os
import re
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_build")

TEST_CASES = [
    "W gradients are bitwise identical across P in {1,2,4,8}",
    "training reduces the loss on a separable toy dataset",
    "identical seeds and P give bitwise-identical loss sequences",
    "training with overlap on equals overlap off bitwise",
    "distributed trajectories are bitwise identical to single-worker",
]


def block(text, start):
    """Text from `start` (a signature or TEST_CASE(...)) through the brace closing its body: the first '{'
    after the parenthesised list that follows `start`."""
    p, q = text.index("(", start), text.index("{", start)
    if p < q:  # skip the parameter list (a TEST_CASE name may contain braces)
        depth = 0
        for q in range(p, len(text)):
            depth += {"(": 1, ")": -1}.get(text[q], 0)
            if depth == 0:
                break
    i = text.index("{", q)
    depth = 0
    for j in range(i, len(text)):
        depth += {"{": 1, "}": -1}.get(text[j], 0)
        if depth == 0:
            return text[start:j + 1]
    raise ValueError("unbalanced braces")


def main():
    ref = sys.argv[1] if len(sys.argv) > 1 else "/root/reference"
    main_cpp = os.path.join(ref, "proj", "tools", "main.cpp")
    test_gcn = os.path.join(ref, "proj", "tests", "test_gcn.cpp")
    if not (os.path.exists(main_cpp) and os.path.exists(test_gcn)):
        print("extract.py: reference not present (build container only)", file=sys.stderr)
        return 3
    os.makedirs(OUT, exist_ok=True)
    src = open(main_cpp).read()
    flags = block(src, src.index("struct CommonFlags {")) + ";\n"
    run_train = block(src, src.index("template <class S>\nint run_train("))
    with open(os.path.join(OUT, "run_train.inc"), "w") as f:
        f.write(f"// extracted from {main_cpp} at build time (not committed)\n{flags}\n{run_train}\n")
    t = open(test_gcn).read()
    helpers = [block(t, t.index(sig)) for sig in (
        "Dataset<double> community_dataset(", "Dataset<double> random_dataset(", "GcnConfig make_cfg(")]
    cases = [block(t, t.index(f'TEST_CASE("{name}")')) for name in TEST_CASES]
    body = "\n\n".join(helpers) + "\n\n" + "\n\n".join(cases)
    body = re.sub(r"\bdouble\b", "float", body)
    with open(os.path.join(OUT, "test_gcn_cases.inc"), "w") as f:
        f.write(f"// extracted from {test_gcn} at build time (not committed); S = double -> float\n{body}\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
