"""Model JSON and dataset CSV formats (reference nn.py:190-220,
training.py:140-152), byte-compatible with the reference's files so models and
datasets move between the two packages unchanged."""

from __future__ import annotations

import json

import numpy as np

from .fields import MlpModel, MlpSpec


def model_to_json(model: MlpModel) -> str:
    """Same document as the reference (nn.py:190-199): spec + theta as floats."""
    theta = model.theta.detach().cpu().numpy().astype(np.float64)
    doc = {
        "spec": {
            "layer_widths": list(model.spec.layer_widths),
            "activation": model.spec.activation,
            "time_input": model.spec.time_input,
        },
        "theta": [float(x) for x in theta],
    }
    return json.dumps(doc)


def model_from_json(text: str, dtype: str = "f64") -> MlpModel:
    doc = json.loads(text)
    spec = MlpSpec(tuple(doc["spec"]["layer_widths"]), doc["spec"]["activation"],
                   bool(doc["spec"]["time_input"]), dtype)
    return MlpModel(spec, np.asarray(doc["theta"], dtype=np.float64))


def save_model(model: MlpModel, path):
    with open(path, "w") as fh:
        fh.write(model_to_json(model))


def load_model(path, dtype: str = "f64") -> MlpModel:
    with open(path) as fh:
        return model_from_json(fh.read(), dtype)


def write_dataset_csv(dataset, path):
    """Header ``t,u1,..,uN`` then one row per sample time, %.17g (training.py:140-147)."""
    n = dataset.observations[0].shape[0]
    header = "t," + ",".join(f"u{i + 1}" for i in range(n))
    with open(path, "w") as fh:
        fh.write(header + "\n")
        for t, row in zip(dataset.times, dataset.observations):
            cells = [f"{t:.17g}"] + [f"{x:.17g}" for x in row]
            fh.write(",".join(cells) + "\n")


def read_dataset_csv(path):
    from .training import Dataset
    rows = np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)
    return Dataset(times=rows[:, 0], observations=[r for r in rows[:, 1:]])
