"""The host worker pool of the host-tier streamer (csrc/pool.h: pageable -> pinned bounce copies,
P:213) under ThreadSanitizer: 200 parallel copies and parallel_for jobs of varying widths, checked
byte for byte, with no data race reported.  CPU only."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_copy_pool_threadsanitizer(tmp_path):
    exe = str(tmp_path / "pool_tsan")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-g", "-fsanitize=thread", "-pthread",
                        "-I", os.path.join(ROOT, "paper_2510_20878_b200", "csrc"),
                        os.path.join(ROOT, "tests", "csrc", "pool_tsan.cpp"), "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    env = dict(os.environ, TSAN_OPTIONS="halt_on_error=1 second_deadlock_stack=1")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300, env=env)
    assert "ThreadSanitizer" not in r.stderr, r.stderr[-4000:]
    assert r.returncode == 0 and "0 mismatches" in r.stdout, r.stdout + r.stderr[-2000:]
