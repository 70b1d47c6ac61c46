"""Golden output of the reference's acceptance gate, criteria 1-9
(/root/reference/proj/tests/acceptance/acceptance.cpp:85-391), from the
UNMODIFIED gate built by oracle/Makefile (oracle/_ref/acceptance_cpu). Run
here, from the repo root:
    make -C oracle gpuseam && python tests/golden/make_golden_acceptance.py
Criterion 10 needs the reference CLI (not buildable: no CLI11) and criterion
11 fails on the reference itself (quirk Q1); both are out.
The GPU suite runs the same gate with every run_simulation call on the B200
(oracle/_ref/acceptance_gpu) and must print these lines byte for byte."""
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
CRITERIA = list(range(1, 10))


def main():
    out = {}
    for i in CRITERIA:
        r = subprocess.run([os.path.join(REPO, "oracle", "_ref", "acceptance_cpu"), str(i)],
                           cwd=REPO, capture_output=True, text=True, check=True)
        out[str(i)] = r.stdout
        print(r.stdout, end="")
    with open(os.path.join(HERE, "acceptance.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
