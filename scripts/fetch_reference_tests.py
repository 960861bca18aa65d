"""Fetch the reference's own tests for the drop-in boundary into
tests/refsuite/ (git-ignored, so reference sources stay out of the history;
gpurun still ships them to the GPU box).  They run UNMODIFIED against this
package: tests/conftest.py aliases the module names they import (embcache,
embcache.runtime, embcache.neural.model, ...) to paper_2511_08568_b200 and
provides their conftest helpers.  SURVEY.md §8(b) names the callers:
test_runtime.py, test_model.py, test_cache_sim.py; test_labeler.py and
test_trace.py cover the labeler and the trace formats built here too.

    python scripts/fetch_reference_tests.py   (also run by __graft_entry__.build())
"""
import os
import shutil
import sys

SRC = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(ROOT, "tests", "refsuite")
FILES = ("test_runtime.py", "test_model.py", "test_cache_sim.py", "test_labeler.py",
         "test_trace.py")


def fetch() -> int:
    if not os.path.isdir(SRC):
        return 0
    os.makedirs(DST, exist_ok=True)
    n = 0
    for f in FILES:
        src = os.path.join(SRC, f)
        if os.path.exists(src):
            shutil.copyfile(src, os.path.join(DST, f))
            n += 1
    return n


if __name__ == "__main__":
    print(f"fetched {fetch()} reference test files into {DST}", file=sys.stderr)
