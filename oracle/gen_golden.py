"""Generate the committed golden fixtures under tests/golden/ by running the
REFERENCE itself (oracle/_ref/libref_latq.so, the unmodified latq sources
compiled in place).  Run in the build container (needs /root/reference):

    make -C oracle ref oracle && python -m oracle.gen_golden

Fixtures (small; the GPU box never needs /root/reference):
  <name>.qshp        artifact bytes from the reference producer
  <name>.x.npy       inputs (f64 values exactly representable in f32)
  <name>.y.npy       latq::infer(artifact, x) from the reference (f64)
  kat.json           known answers pinned by the reference's own tests
"""
from __future__ import annotations

import json
import os

import numpy as np

from oracle.refpy import Ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden")

# name, m, n, bits, seed, producer ("hi" = H=I route; "psd" = quantize_layer with a random PSD H),
# transform (0 = rht, 1 = rfft)
CASES = [
    ("e8p2_64x64", 64, 64, 2, 0, "psd", 0),
    ("rvq3_64x64", 64, 64, 3, 1, "psd", 0),
    ("rvq4_64x64", 64, 64, 4, 2, "psd", 0),
    ("e8p2_128x256", 128, 256, 2, 3, "hi", 0),
    ("rvq3_256x128", 256, 128, 3, 4, "hi", 0),
    ("rvq4_128x128", 128, 128, 4, 5, "hi", 0),
    ("e8p2_96x160", 96, 160, 2, 6, "hi", 0),     # q = 12 (96 = 8*12), q = 20 (160 = 8*20)
    ("rvq3_56x112", 56, 112, 3, 7, "hi", 0),     # q = 28 (56 = 2*28, 112 = 4*28)
    ("e8p2_1024x1024", 1024, 1024, 2, 8, "hi", 0),
    # rfft transform (rfft.cpp; DFT lengths m/2, n/2)
    ("rfft2_64x64", 64, 64, 2, 10, "psd", 1),
    ("rfft3_56x112", 56, 112, 3, 11, "hi", 1),   # 28 = 4*7, 56 = 8*7
    ("rfft4_96x160", 96, 160, 4, 12, "hi", 1),
    ("rfft2_30x64", 30, 64, 2, 13, "hi", 1),     # odd left length 15
    ("rfft2_344x512", 344, 512, 2, 14, "hi", 1),  # 172 = 4*43
]


def make_case(ref: Ref, m, n, bits, seed, producer, transform=0) -> bytes:
    if producer == "hi":
        return ref.quantize_hi(m, n, bits, seed, transform=transform)
    rng = np.random.default_rng(1000 + seed)
    w = ref.gen_weights(m, n, ref.substream_seed(seed, 10))
    x = rng.standard_normal((n, 2 * n))
    h = x @ x.T / (2 * n)
    return ref.quantize_layer(w, h, bits, seed, transform=transform)


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    ref = Ref()
    index = []
    for name, m, n, bits, seed, producer, transform in CASES:
        art = make_case(ref, m, n, bits, seed, producer, transform)
        assert ref.roundtrip(art) == art
        rng = np.random.default_rng(seed)
        x = rng.standard_normal((4, n)).astype(np.float32).astype(np.float64)
        x[3] /= np.linalg.norm(x[3])  # unit input, as acceptance.cpp:414-416
        y = ref.infer(art, x)
        with open(os.path.join(OUT, f"{name}.qshp"), "wb") as f:
            f.write(art)
        np.save(os.path.join(OUT, f"{name}.x.npy"), x)
        np.save(os.path.join(OUT, f"{name}.y.npy"), y)
        index.append({"name": name, "m": m, "n": n, "bits": bits, "seed": seed, "producer": producer,
                      "transform": transform, "bytes": len(art)})
    d, p = ref.e8p_tables()
    kat = {
        # test_e8p.cpp:72-85
        "e8p_row21": d[21].tolist(),
        "e8p_decode_0x1597": ref.e8p_decode(0x1597).tolist(),
        # test_e8p.cpp:66-69
        "e8p_odd_rows": int(p.sum()),
        "e8p_doubled": d.tolist(),
        "e8p_odd_parity": p.tolist(),
        # test_codebooks.cpp:49-64 (e8-1bit rows 0, 1, 240, 241) + whole table
        "e8_1bit": [ref.codebook_decode("e8-1bit", c).tolist() for c in range(256)],
        # test_hadamard.cpp:64-84
        "plans": {str(n): list(ref.plan_hadamard(n)) for n in (1, 4, 12, 20, 24, 28, 56, 4096, 8192, 28672)},
        "bases": {str(q): ref.hadamard_base(q).tolist() for q in (4, 12, 20, 28)},
        # had_apply on fixed vectors (forward and transpose)
        "had_apply": [],
        # sign vectors from the reference RNG (bitpack.cpp:11-15)
        "signs_seed5_n13": ref.random_signs(13, 5).tolist(),
        "cases": index,
    }
    for n in (4, 12, 20, 24, 28, 40, 56, 112, 4096):
        x = np.random.default_rng(n).standard_normal(n)
        kat["had_apply"].append({"n": n, "x": x.tolist(), "fwd": ref.had_apply(x).tolist(),
                                 "bwd": ref.had_apply(x, True).tolist()})
    # rfft_apply (rfft.cpp:39-71) on fixed vectors with reference phases
    # (PhaseVector::random, bitpack.cpp:42-53), lengths as test_rfft.cpp
    kat["rfft_apply"] = []
    for n in (2, 8, 10, 64, 100, 344):
        ph = ref.random_phases(n, 7 * n + 1)
        x = np.random.default_rng(n + 3).standard_normal(n)
        kat["rfft_apply"].append({"n": n, "phases": ph.tolist(), "x": x.tolist(),
                                  "fwd": ref.rfft_apply(ph, x).tolist(), "bwd": ref.rfft_apply(ph, x, True).tolist()})
    with open(os.path.join(OUT, "kat.json"), "w") as f:
        json.dump(kat, f)
    print(f"wrote {len(index)} cases + kat.json to {OUT}")


if __name__ == "__main__":
    main()
