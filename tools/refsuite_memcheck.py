"""The reference's own test files against this package under compute-sanitizer memcheck, torch's caching
allocator off (developer tool; needs baseline/_ref/tests or /root/reference: tools/stage_reference_tests.sh)."""
import os, shutil, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_reference_suite as T
src = T.find_tests()
assert src, "reference tests not staged"
with tempfile.TemporaryDirectory() as td:
    for f in T.FILES:
        shutil.copy(os.path.join(src, f), os.path.join(td, f))
    open(os.path.join(td, "conftest.py"), "w").write(T.CONFTEST % ROOT)
    env = dict(os.environ, HYPOTHESIS_STORAGE_DIRECTORY=os.path.join(td, ".hyp"), NUMBA_CACHE_DIR=os.path.join(td, ".numba"),
               PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    r = subprocess.run(["compute-sanitizer", "--tool", "memcheck", "--print-limit", "3", sys.executable, "-m", "pytest", "-q", "-p",
                        "no:cacheprovider", "--rootdir", td, "-c", "/dev/null", "-rfE", "--tb=line", *T.FILES],
                       cwd=td, env=env, capture_output=True, text=True, timeout=3000)
out = r.stdout + r.stderr
open(os.path.join(ROOT, "gpurun_out", "refsuite_memcheck.log"), "w").write(out)
for l in out.splitlines():
    if "ERROR SUMMARY" in l or " passed" in l or "Invalid" in l or l.startswith("FAILED"):
        print(l[:200])
