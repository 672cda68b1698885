"""Golden training runs of the REFERENCE Trainer (lpxmc.trainer, imported from
/root/reference in the build container) that pin the restated training loop
oracle/lpxmc_trainer_oracle.py.  Writes trainer_golden.npz next to this file.

    python tests/golden/make_trainer_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# tests/conftest.py of the reference: the frozen EASY benchmark
EASY_SPEC = dict(num_samples=640, num_features=32, num_labels=32, mean_labels=1.0, min_labels=1, noise=0.05, seed=7)
EASY_CFG = dict(hidden=64, embed_dim=32, head_lr=0.3, encoder_lr=3e-3, epochs=25, batch_size=32, chunks=1, seed=1)

RUNS = {
    # name: (config overrides, epochs run)
    "fp32": ({}, 2),
    "e4m3sr": ({"head_format": "e4m3", "head_rounding": "stochastic", "chunks": 2, "warmup_steps": 5,
                "head_weight_decay": 1e-4}, 1),
    "bf16rtn": ({"head_format": "bf16", "head_rounding": "nearest", "grad_clip": 1.0}, 1),
    "frozen": ({"head_lr": 0.0}, 1),
}


def main():
    sys.path.insert(0, REF)
    from lpxmc.data import SyntheticSpec, generate_synthetic
    from lpxmc.trainer import TrainConfig, Trainer

    ds = generate_synthetic(SyntheticSpec(**EASY_SPEC))
    out = {"ds_labels_flat": np.concatenate(ds.labels), "ds_labels_len": np.array([len(l) for l in ds.labels]),
           "ds_values": np.stack(ds.values)}
    for name, (over, epochs) in RUNS.items():
        cfg = TrainConfig(**{**EASY_CFG, **over})
        t = Trainer(ds, cfg)
        mean_g = []
        step = t.step

        def logged(batch_idx, probe=None, input_probe=None, _step=step):
            g = _step(batch_idx, probe=probe, input_probe=input_probe)
            mean_g.append(g)
            return g
        t.step = logged
        hist = [t.run_epoch() for _ in range(epochs)]
        out[f"{name}_mean_g"] = np.array(mean_g)
        out[f"{name}_p_at"] = np.array([[h["p_at_1"], h["p_at_3"], h["p_at_5"]] for h in hist])
        out[f"{name}_head_w"] = t.head.weights.values.copy()
        for pn, p in t.encoder.params.items():
            out[f"{name}_enc_{pn}"] = p.values.copy()
        out[f"{name}_eval_idx"] = t.eval_idx
    path = os.path.join(HERE, "trainer_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
