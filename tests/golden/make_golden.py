"""Generate the golden fixtures that pin the oracle to the reference (run in the
build container, where /root/reference exists; the fixtures are committed and
nothing at test time reads /root/reference).

    python tests/golden/make_golden.py

Fixtures (tests/golden/reference_conventions.npz):
* uniforms_*      gbsemu.sampler._stream_uniforms(seed, start, count, M)  (sampler.py:109-125)
* exact_*         gbsemu.sampler.exact_reference_sampler on a 4-mode random instance:
                  its distribution p, uniforms u and drawn codes (sampler.py:686-703) —
                  pins the inverse-CDF rule the MPS draw uses
* coherent_*      gbsemu.gaussian.vacuum_overlap of displaced vacua (gaussian.py:231-253):
                  single mode |<0|D(a)|0>|^2 and an M-mode product of them
"""

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from gbsemu import gaussian as g  # noqa: E402
from gbsemu import sampler as sp  # noqa: E402

HBAR = 2.0
out = {}

cases = [(0, 0, 200, 8), (7, 100, 300, 16), (123456789, 63, 3, 64), (2**63 + 5, 1000, 130, 5), (0, 0, 1, 1)]
for j, (seed, start, count, M) in enumerate(cases):
    out[f"uniforms_{j}_args"] = np.array([seed, start, count, M], dtype=np.uint64)
    out[f"uniforms_{j}"] = sp._stream_uniforms(seed, start, count, M)

inst, _ = g.random_instance(M=4, k=2, eta=0.7, r_max=1.2, seed=11)
cfg = sp.SamplerConfig(N=5000, method="exact_reference", seed=3)
batch = sp.exact_reference_sampler(inst, cfg)
codes = (batch.bitstrings.astype(np.int64) << np.arange(3, -1, -1)).sum(axis=1)
out["exact_p"] = g.brute_force_distribution(inst)
out["exact_u"] = sp._stream_uniforms(3, 0, 5000, 1)[:, 0]
out["exact_codes"] = codes

rng = np.random.default_rng(5)
alphas = (rng.standard_normal(12) + 1j * rng.standard_normal(12)) * 0.6
vac = []
for a in alphas:
    mu = np.sqrt(2 * HBAR) * np.array([a.real, a.imag])
    vac.append(g.vacuum_overlap(np.eye(2), mu, hbar=HBAR))
out["coherent_alpha"] = alphas
out["coherent_vacuum_prob"] = np.array(vac)
# 5-mode product of displaced vacua (xxpp ordering, gaussian.py:1-13)
Mm = 5
am = alphas[:Mm] * 0.5
mu = np.sqrt(2 * HBAR) * np.concatenate([am.real, am.imag])
out["coherent_multimode_alpha"] = am
out["coherent_multimode_vacuum_prob"] = np.array(g.vacuum_overlap(np.eye(2 * Mm), mu, hbar=HBAR))

# the reference's sample text format (sampler.py:772-778) for a small click batch
import tempfile  # noqa: E402

rng = np.random.default_rng(9)
bits = (rng.random((7, 6)) < 0.4).astype(np.uint8)
sb = sp.SampleBatch(M=6, N=7, bitstrings=bits, method="mps", K=0, seed=11)
with tempfile.TemporaryDirectory() as d:
    sp.save_samples_text(Path(d) / "s.txt", sb)
    out["text_bits"] = bits
    out["text_bytes"] = np.frombuffer((Path(d) / "s.txt").read_bytes(), dtype=np.uint8)

np.savez_compressed(Path(__file__).with_name("reference_conventions.npz"), **out)
print("wrote", len(out), "arrays")
