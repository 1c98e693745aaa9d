"""SGRPOCK1 wire format (src/tinylm.cpp:14-105). Golden files were written by
the compiled reference (tests/golden/make_golden.py::checkpoint_fixture). The library parses
the header on the host (no GPU), loads a checkpoint straight into the device weights, and
writes the online-learned draft back in the reference's exact byte layout."""
import json
import os
import shutil

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _cfg():
    return json.load(open(os.path.join(GOLD, "ckpt.json")))["config"]


def test_header_parse_matches_reference_files(tmp_path):
    from paper_2509_21792_b200 import capi
    cfg = _cfg()
    for name, kind in (("ckpt_target.bin", "target"), ("ckpt_draft.bin", "draft")):
        info = capi.checkpoint_info(os.path.join(GOLD, name))
        assert info["kind"] == kind
        for k, v in cfg.items():
            assert info[k] == v, k
        k2, p = O.load_checkpoint(os.path.join(GOLD, name))
        assert k2 == kind and info["param_count"] == p.flat.size
    assert capi.checkpoint_info(os.path.join(GOLD, "ckpt_draft.bin"))["draft_layers"] == 1
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTACKPT" + bytes(8))
    with pytest.raises(RuntimeError):
        capi.checkpoint_info(str(bad))
    with pytest.raises(RuntimeError):
        capi.checkpoint_info(str(tmp_path / "missing.bin"))


@pytest.mark.gpu
def test_device_load_and_save_roundtrip(tmp_path):
    from tests.gpu_common import capi as load_capi
    c = load_capi()
    cfg = O.ModelConfig(**_cfg())
    _, tgt = O.load_checkpoint(os.path.join(GOLD, "ckpt_target.bin"))
    _, dr = O.load_checkpoint(os.path.join(GOLD, "ckpt_draft.bin"))
    a = c.Engine(cfg, 1, 0, 4, 64, 4, 3)
    assert a.load_checkpoint(os.path.join(GOLD, "ckpt_target.bin")) == "target"
    assert a.load_checkpoint(os.path.join(GOLD, "ckpt_draft.bin")) == "draft"
    b = c.Engine(cfg, 1, 0, 4, 64, 4, 3)
    b.upload_target(tgt.flat)
    b.upload_draft(dr.flat)
    # the draft master is the file payload, bit for bit
    assert np.array_equal(a.download_draft(), dr.flat)
    # the target behaves exactly like the host-uploaded copy
    toks = [3, 9, 17, 33, 2, 60]
    la, ha = a.forward_target(0, toks, list(range(len(toks))))
    lb, hb = b.forward_target(0, toks, list(range(len(toks))))
    assert np.array_equal(la, lb) and np.array_equal(ha, hb)
    # writing the draft back reproduces the reference's file byte for byte
    out = tmp_path / "draft.bin"
    a.save_draft_checkpoint(str(out))
    assert out.read_bytes() == open(os.path.join(GOLD, "ckpt_draft.bin"), "rb").read()
    # a checkpoint of another shape is refused
    other = O.ModelConfig(cfg.vocab_size, cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.max_seq_len + 8, 5)
    e3 = c.Engine(other, 1, 0, 4, 64, 4, 3)
    with pytest.raises(ValueError):
        e3.load_checkpoint(os.path.join(GOLD, "ckpt_target.bin"))
    trunc = tmp_path / "trunc.bin"
    shutil.copy(os.path.join(GOLD, "ckpt_target.bin"), trunc)
    with open(trunc, "r+b") as f:
        f.truncate(1000)
    with pytest.raises(RuntimeError):
        a.load_checkpoint(str(trunc))
