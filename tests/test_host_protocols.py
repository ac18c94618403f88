"""Host-side protocols of the pinned-memory hand-offs, exercised on the CPU with fake GPU producers
(SURVEY.md §4 layer 1 "the ring protocol with a CPU fake producer ... under ThreadSanitizer"; test
idea from SPEC.md:121-153, not its program): the staged host tier's chunk-claim protocol
(csrc/staging.cu compiled in unchanged) and the IO rings' SQ/CQ hand-off (csrc/cache.cu's io_worker
compiled in unchanged).  Each harness checks every byte it produced against its source, and the
-fsanitize=thread builds check the memory ordering of the protocols.  No GPU, no CUDA runtime calls.
"""
import json
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
NATIVE = os.path.join(HERE, "native")
CUDA_INC = "/usr/local/cuda/include"


def _build(src: str, out: str, tsan: bool) -> str:
    exe = os.path.join("/tmp", f"{out}{'_tsan' if tsan else ''}_{os.getpid()}")
    flags = ["-O1", "-g", "-fsanitize=thread"] if tsan else ["-O2"]
    subprocess.check_call(["g++", *flags, "-std=c++17", "-x", "c++", f"-I{CUDA_INC}", "-pthread", "-o", exe,
                           os.path.join(NATIVE, src)])
    return exe


def _run(exe: str, *args) -> dict:
    r = subprocess.run([exe, *map(str, args)], capture_output=True, text=True, timeout=600,
                       env={**os.environ, "TSAN_OPTIONS": "halt_on_error=1 exitcode=66"})
    assert r.returncode == 0, (r.returncode, r.stdout[-2000:], r.stderr[-4000:])
    assert "ThreadSanitizer" not in r.stderr, r.stderr[-4000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module", params=[False, True], ids=["plain", "tsan"])
def stager(request):
    return _build("stager_harness.cpp", "stager_harness", request.param), request.param


@pytest.mark.parametrize("ctx,batches,n_host,workers,gpu,frac,steal,reserve,reserve_us",
                         [(3, 40, 5000, 4, 4, 1.0, 100, 0, 0), (4, 30, 3000, 6, 2, 0.5, 100, 0, 0),
                          (2, 60, 700, 3, 3, 1.0, 0, 0, 0), (1, 50, 64, 2, 1, 1.0, 1000, 0, 0),
                          (3, 20, 20000, 8, 6, 0.6, 20, 0, 0), (3, 30, 5000, 4, 4, 1.0, 100, 0.7, 200),
                          (2, 30, 3000, 1, 4, 0.7, 50, 0.7, 5), (4, 20, 8000, 6, 3, 0.8, 100, 0.8, 1000)])
def test_stager_chunk_protocol(stager, ctx, batches, n_host, workers, gpu, frac, steal, reserve, reserve_us):
    """Every host-list row of every batch reaches the output exactly as its source row, whatever
    mix of zero-copy and staged chunks the race produced; staged chunks were used."""
    exe, tsan = stager
    if tsan:
        batches = max(5, batches // 3)
    r = _run(exe, ctx, batches, n_host, workers, gpu, frac, steal, reserve, reserve_us)
    assert r["bad_rows"] == 0
    assert r["rows_gpu"] + r["rows_staged_used"] > 0
    assert r["rows_staged_by_cpu"] >= r["rows_staged_used"]


@pytest.fixture(scope="module", params=[False, True], ids=["plain", "tsan"])
def rings(request):
    return _build("ring_harness.cpp", "ring_harness", request.param), request.param


@pytest.mark.parametrize("rings_n,depth,producers,requests,fault", [(2, 2, 2, 1000, 0), (4, 8, 3, 3000, 0),
                                                                    (1, 4, 1, 500, 0), (3, 4, 2, 1000, 137)])
def test_io_ring_conservation(rings, rings_n, depth, producers, requests, fault):
    """SQ/CQ rings with the real host IO workers (cache.cu io_worker) and CPU fake producers in the
    GPU kernel's role: the multiset of completed requests equals the submitted one (every request
    completed exactly once, SPEC.md:150 idea), every staged row holds the right file bytes, ring
    depth 2 forces wrap-around and back-pressure, and an injected read fault is reported for exactly
    that request."""
    exe, tsan = rings
    r = _run(exe, rings_n, depth, producers, requests if not tsan else requests // 2, fault)
    assert r["bad_bytes"] == 0 and r["missing"] == 0 and r["duplicates"] == 0
    assert r["completed"] == r["submitted"]
    assert r["io_errors"] == (1 if fault else 0)
