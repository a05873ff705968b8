"""Checkpoint / snapshot files from the device state:
CKCHKPT1 and CKSNAP1 (io.hpp:344-430) written by the Python twin from the
device-packed records (ckg_pack_records) against the reference engine's own
writers (oracle/_ref) on the same state, and restart parity."""
import os

import numpy as np
import pytest

from oracle import bind
from paper_2412_10399_b200.scene import IoError, seed_particles
from tests.gpu_util import gpu_sim, match_by_tag, tag_volumes
from tests.util import small_scene

pytestmark = pytest.mark.gpu


def _ref_io_available(ref, tmp_path):
    return ref.write_checkpoint(tmp_path / "probe.ckpt") != 5


@pytest.mark.parametrize("model", ["fixed_corotated", "j_fluid"])
def test_files_byte_identical_to_reference(tmp_path, model):
    cfg = small_scene(model=model, res=32, bc="slip" if model == "j_fluid" else "sticky")
    p = seed_particles(cfg)
    ref = bind.Ref(cfg, p)
    if not _ref_io_available(ref, tmp_path):
        pytest.skip("reference shim built without io.hpp")
    sim = gpu_sim(cfg, p)
    for kind in ("ckpt", "snap", "txt"):
        r, g = tmp_path / f"ref.{kind}", tmp_path / f"gpu.{kind}"
        if kind == "ckpt":
            assert ref.write_checkpoint(r) == 0
            sim.write_checkpoint(g)
        else:
            assert ref.write_snapshot(r, 7, binary=(kind == "snap")) == 0
            sim.write_snapshot(g, 7, binary=(kind == "snap"))
        assert r.read_bytes() == g.read_bytes(), kind


def test_checkpoint_after_steps_and_restart(tmp_path):
    cfg = small_scene(res=32)
    p = tag_volumes(seed_particles(cfg))
    ref = bind.Ref(cfg, p)
    sim = gpu_sim(cfg, p)
    for _ in range(8):
        dt = ref.cfl_dt(1.0)
        assert ref.step(dt)[0] == 0
        sim.step(dt)
    if _ref_io_available(ref, tmp_path):
        assert ref.write_checkpoint(tmp_path / "ref.ckpt") == 0
        sim.write_checkpoint(tmp_path / "gpu.ckpt")
        a, b = (tmp_path / "ref.ckpt").read_bytes(), (tmp_path / "gpu.ckpt").read_bytes()
        assert len(a) == len(b)
        hdr = 8 + 4 + 8 + 4 + 8 + 8 + 8  # magic scalar step frame time eps count (double)
        assert a[:24] == b[:24]  # magic, scalar width, step, frame
        # same particle order (sorted by the same keys); values agree to round-off
        ra = np.frombuffer(a, dtype=np.dtype([("f", "<f8", 27), ("m", "<u4")]), offset=hdr)
        rb = np.frombuffer(b, dtype=np.dtype([("f", "<f8", 27), ("m", "<u4")]), offset=hdr)
        assert np.array_equal(ra["f"][:, 26], rb["f"][:, 26])  # volume0 tags: identical order
        assert np.max(np.abs(ra["f"] - rb["f"])) <= 1e-9
    # restart: read back, continue next to the uninterrupted run
    sim.write_checkpoint(tmp_path / "s.ckpt")
    again = gpu_sim(cfg, p)
    again.read_checkpoint(tmp_path / "s.ckpt")
    assert again.step_count() == sim.step_count() and again.time() == sim.time()
    again.write_checkpoint(tmp_path / "again.ckpt")
    assert (tmp_path / "again.ckpt").read_bytes() == (tmp_path / "s.ckpt").read_bytes()
    for _ in range(5):
        dt = sim.cfl_dt(1.0)
        assert dt == again.cfl_dt(1.0)
        sim.step(dt)
        again.step(dt)
    x, y = match_by_tag(sim.particles(), again.particles())
    assert np.max(np.abs(x["x"] - y["x"])) <= 1e-12


def test_read_checkpoint_errors(tmp_path):
    cfg = small_scene(res=32)
    sim = gpu_sim(cfg, seed_particles(cfg))
    (tmp_path / "bad").write_bytes(b"NOTACKPT" + b"\0" * 64)
    with pytest.raises(IoError, match="not a checkpoint file"):
        sim.read_checkpoint(tmp_path / "bad")
    sim.write_checkpoint(tmp_path / "ok")
    data = (tmp_path / "ok").read_bytes()
    (tmp_path / "short").write_bytes(data[: len(data) - 100])
    with pytest.raises(IoError, match="truncated checkpoint particle data"):
        sim.read_checkpoint(tmp_path / "short")
