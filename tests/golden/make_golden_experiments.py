"""Golden outputs of the reference's experiment commands (run / compare /
sweep through its own C ABI, kvadmit.h:58-78, unmodified sources in
oracle/_ref/libkvref.so) for every preset that defines them. Run here:
    python tests/golden/make_golden_experiments.py
  experiments.json: per (preset, command): rendered text, and every file the
  command wrote (path relative to its directory -> sha256)."""
import ctypes as C
import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from tests.helpers import ref_lib  # noqa: E402

PRESETS = "/root/reference/proj/configs"
JOBS = [("smoke", "compare"), ("ample", "compare"), ("thrash", "compare"), ("thrash", "sweep"),
        ("sweep-sensitivity", "sweep"), ("sweep-sensitivity-ulow", "sweep"), ("smoke", "run"),
        ("thrash", "run")]


def tree_hashes(d):
    out = {}
    for root, _, files in os.walk(d):
        for f in files:
            p = os.path.join(root, f)
            out[os.path.relpath(p, d)] = hashlib.sha256(open(p, "rb").read()).hexdigest()
    return dict(sorted(out.items()))


def main():
    lib = ref_lib()
    lib.kva_scenario_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    for f in ("kva_cmd_compare", "kva_cmd_sweep"):
        getattr(lib, f).argtypes = [C.c_void_p, C.c_char_p, C.c_uint, C.POINTER(C.c_void_p)]
    lib.kva_cmd_run.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]
    lib.kva_text_free.argtypes = [C.c_void_p]
    lib.kva_last_error.restype = C.c_char_p
    out = {}
    for preset, cmd in JOBS:
        sc = C.c_void_p()
        assert lib.kva_scenario_load(os.path.join(PRESETS, preset + ".toml").encode(),
                                     C.byref(sc)) == 0, lib.kva_last_error()
        with tempfile.TemporaryDirectory() as root:
            text = C.c_void_p()
            if cmd == "run":
                rc = lib.kva_cmd_run(sc, root.encode(), C.byref(text))
            else:
                rc = getattr(lib, "kva_cmd_" + cmd)(sc, root.encode(), 1, C.byref(text))
            assert rc == 0, lib.kva_last_error()
            rendered = C.cast(text, C.c_char_p).value.decode()
            lib.kva_text_free(text)
            sub = os.listdir(root)
            assert len(sub) == 1
            out[f"{preset}/{cmd}"] = dict(dir=sub[0], files=tree_hashes(os.path.join(root, sub[0])),
                                          text=rendered.replace(root, "<root>"))
        print(preset, cmd, len(out[f"{preset}/{cmd}"]["files"]), "files")
    with open(os.path.join(HERE, "experiments.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
