"""Small synthetic network bodies for parity tests (CPU + GPU)."""
import numpy as np


def conv_spec(rng, in_c, out_c, k, stride, pad, ta=(0.5, 0.9)):
    K = in_c * k * k
    # variance-normalising folded-BN gain so every activation level occurs
    gain = (rng.uniform(0.8, 1.2, out_c) / np.sqrt(K)).astype(np.float32)
    bias = (rng.standard_normal(out_c) * 0.2).astype(np.float32)
    return dict(in_c=in_c, out_c=out_c, k=k, stride=stride, pad=pad,
                weights=rng.integers(-1, 2, (out_c, K)).astype(np.int8),
                ta=ta, tw=(1.0, 1.0), gain=gain, bias=bias, out_scale=1.0)


def tiny_body(seed=0, n=2, c=16, h=12, w=12):
    rng = np.random.default_rng(seed)
    blocks = [
        dict(convs=[conv_spec(rng, c, c, 3, 1, 1), conv_spec(rng, c, c, 3, 1, 1, (0.45, 0.8))]),
        dict(convs=[conv_spec(rng, c, 2 * c, 3, 2, 1), conv_spec(rng, 2 * c, 2 * c, 3, 1, 1)],
             down=conv_spec(rng, c, 2 * c, 1, 2, 0)),
        dict(convs=[conv_spec(rng, 2 * c, c, 1, 1, 0), conv_spec(rng, c, c, 3, 1, 1),
                    conv_spec(rng, c, 2 * c, 1, 1, 0)]),
    ]
    x = np.abs(rng.standard_normal(n * c * h * w)).astype(np.float32)
    return blocks, (n, c, h, w), x
