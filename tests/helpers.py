"""Shared test helpers: golden-vector decoding."""
import numpy as np


def f32_from_bits(bits) -> np.ndarray:
    return np.asarray(bits, dtype=np.uint32).view(np.float32)


def bits_of(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def hex_bytes(s: str) -> np.ndarray:
    return np.frombuffer(bytes.fromhex(s), dtype=np.uint8).copy()


def case_inputs(oracle, case):
    """Re-generate a hot_path case's inputs with the oracle RNG (pinned against the
    inputs the reference emitted where they are present)."""
    r = oracle.rng(case["seed"])
    a = oracle.gaussian_fill(r, (case["m"], case["k"]), 1.0)
    w = oracle.gaussian_fill(r, (case["n"], case["k"]), case["w_sd"])
    gamma = beta = None
    if case["clip"]:
        gamma = f32_from_bits(case["gamma_bits"])
        beta = f32_from_bits(case["beta_bits"])
    return a, w, gamma, beta
