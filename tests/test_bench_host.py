"""Host-side checks of the benchmark inputs and of bench.py's reference arm
(no GPU): the committed clips are the ones the reference decoder was run on
(bench_8k.json), set 0 of the 8K clip is the reference encoder's output, and
``bench.py --impl reference`` runs the unmodified reference package without
mapping any of this repo's native code."""
import hashlib
import json
import lzma
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

sys.path.insert(0, os.path.join(ROOT, "scripts"))
import make_bench_input as mbi  # noqa: E402


@pytest.fixture(scope="module")
def fixture():
    with open(os.path.join(GOLDEN, "bench_8k.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("cfg", ["c3", "c2"])
def test_committed_clip_sha(fixture, cfg, tmp_path):
    p = mbi.ensure_clip(cfg, str(tmp_path))
    with open(p, "rb") as fh:
        assert hashlib.sha256(fh.read()).hexdigest() == fixture["clips"][cfg]["sha256"]


def test_clip_set0_is_reference_encoder_output(fixture, tmp_path):
    from paper_2208_10859_b200.fileio import VideoReader
    ref = fixture["reference_encoder_set0"]
    assert ref["bench_clip_set0_equal"]
    p = mbi.ensure_clip("c3", str(tmp_path))
    with VideoReader(p) as r:
        m = r.set_meta[0]
        h = r.header
        ext = np.ascontiguousarray(m.extrema, np.float32).tobytes()
    with open(p, "rb") as fh:
        fh.seek(m.payload_offset)
        payload = fh.read(m.payload_length)
    assert hashlib.sha256(payload).hexdigest() == ref["payload_sha256"]
    assert hashlib.sha256(ext).hexdigest() == ref["extrema_sha256"]
    assert (h.width, h.height, h.levels, h.inter_size, h.num_sets, h.stereo) == (
        8192, 8192, 6, 4, 4, True)


def test_display_schedule_walks_the_trajectory():
    traj = mbi.trajectory_table()
    seen = {mbi.display_step(i, 16, 120.0, traj)[1:3] for i in range(64)}
    frames = [mbi.display_step(i, 16, 120.0, traj)[0] for i in range(32)]
    assert len(seen) >= 60          # a new head pose (almost) every step
    assert frames[:16] == list(range(16)) and frames[16:] == list(range(16))


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "wavevid")),
                    reason="reference not installed in baseline/_ref")
def test_reference_arm_runs_reference_without_repo_native(tmp_path):
    """bench.py --impl reference on a small stereo file: the JSON line
    names the reference, and no paper_2208_10859_b200 shared object was
    mapped in the arm's processes."""
    clip = os.path.join(GOLDEN, "golden_stereo.wvv")
    env = dict(os.environ, PYTHONPATH="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--clip", clip, "--steps", "2", "--warmup", "1",
                        "--cache-dir", str(tmp_path)],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["repo_native_loaded"] == []
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert "torch" not in r.stderr
