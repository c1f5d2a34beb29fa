import os
import sys
sys.path.insert(0, "/root/repo")
import tests.test_gpu_gather as T
try:
    T.test_gather_matches_canvas(((40, 36), 2, 2, 0.10, 400), "int8")
    print("GDBG", os.environ.get("PMX_GDBG"), "ok")
except AssertionError as e:
    print("GDBG", os.environ.get("PMX_GDBG"), "mismatch (no crash)")
except Exception as e:
    print("GDBG", os.environ.get("PMX_GDBG"), "ERROR", str(e)[:80])
