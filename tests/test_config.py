"""TrainConfig (reference trainer.py:26-111; its tests/test_trainer.py
config cases): profile defaults, JSON round trip, unknown keys rejected.
CPU only."""

import json

import pytest

from paper_2601_19489_b200.losses import depth_weight_schedule
from paper_2601_19489_b200.trainer import TrainConfig


def test_profiles_resolve_defaults():
    r1 = TrainConfig(round_profile="round1")
    assert r1.max_iters == 6000 and r1.pose_opt and not r1.depth_supervision
    r2 = TrainConfig(round_profile="round2")
    assert r2.max_iters == 15000 and not r2.pose_opt and r2.depth_supervision
    assert depth_weight_schedule(0, r2.max_iters, r2.depth_weight0) == pytest.approx(0.1)
    assert r2.densify_end == int(0.8 * 15000)


def test_config_json_roundtrip(tmp_path):
    cfg = TrainConfig(round_profile="round2", max_iters=123, lambda_=0.3)
    cfg.to_json(tmp_path / "cfg.json")
    back = TrainConfig.from_json(tmp_path / "cfg.json")
    assert back.max_iters == 123 and back.lambda_ == 0.3


def test_config_rejects_unknown_keys(tmp_path):
    (tmp_path / "bad.json").write_text(json.dumps({"max_iters": 10, "not_a_key": 1}))
    with pytest.raises(ValueError, match="not_a_key"):
        TrainConfig.from_json(tmp_path / "bad.json")
