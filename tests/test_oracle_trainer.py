"""The restated training loop (oracle/lpxmc_trainer_oracle.py) reproduces the
reference Trainer's own runs bit for bit (golden vectors from lpxmc itself,
tests/golden/make_trainer_golden.py): dataset, per-step mean |G| (the
divergence proxy), P@1/3/5 after each epoch, final head weights and encoder
parameters -- fp32 head, e4m3 + SR with chunks / warmup / weight decay, bf16
RTN with gradient clipping, and the frozen lr = 0 path."""

import os

import numpy as np
import pytest

from oracle import lpxmc_trainer_oracle as T

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "trainer_golden.npz"))
EASY_SPEC = dict(num_samples=640, num_features=32, num_labels=32, mean_labels=1.0, min_labels=1, noise=0.05, seed=7)
EASY_CFG = dict(hidden=64, embed_dim=32, head_lr=0.3, encoder_lr=3e-3, epochs=25, batch_size=32, chunks=1, seed=1)
RUNS = {
    "fp32": ({}, 2),
    "e4m3sr": ({"head_format": "e4m3", "head_rounding": "stochastic", "chunks": 2, "warmup_steps": 5,
                "head_weight_decay": 1e-4}, 1),
    "bf16rtn": ({"head_format": "bf16", "head_rounding": "nearest", "grad_clip": 1.0}, 1),
    "frozen": ({"head_lr": 0.0}, 1),
}


def test_synthetic_dataset_equals_reference():
    ds = T.generate_synthetic(T.SyntheticSpec(**EASY_SPEC))
    assert np.array_equal(np.concatenate(ds.labels), GOLD["ds_labels_flat"])
    assert np.array_equal(np.stack(ds.values), GOLD["ds_values"])


@pytest.mark.parametrize("name", list(RUNS))
def test_trainer_run_equals_reference(name):
    over, epochs = RUNS[name]
    ds = T.generate_synthetic(T.SyntheticSpec(**EASY_SPEC))
    t = T.Trainer(ds, T.TrainConfig(**{**EASY_CFG, **over}))
    assert np.array_equal(t.eval_idx, GOLD[f"{name}_eval_idx"])
    hist = [t.run_epoch() for _ in range(epochs)]
    assert np.array_equal(np.array(t.mean_g), GOLD[f"{name}_mean_g"])
    assert np.array_equal(np.array([[h["p_at_1"], h["p_at_3"], h["p_at_5"]] for h in hist]), GOLD[f"{name}_p_at"])
    assert np.array_equal(t.head.values.view(np.uint32), GOLD[f"{name}_head_w"].view(np.uint32))
    for pn, p in t.encoder.params.items():
        assert np.array_equal(p.values, GOLD[f"{name}_enc_{pn}"]), pn
