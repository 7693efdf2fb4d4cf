"""Generates the golden fixtures in tests/golden/ by running the REFERENCE
implementation itself (oracle/_ref/libuwbref.so, compiled from
/root/reference/proj/src by oracle/Makefile) on small seeded inputs.

Run here, where /root/reference is mounted:  python tests/golden/make_golden.py
The fixtures pin the oracle restatement (tests/test_oracle.py) and the GPU path
(tests/test_gpu_golden.py) on machines where the reference is not available.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.pyoracle import RefLib  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)


def main():
    ref = RefLib()
    rng = np.random.default_rng(20201120)

    # summed-area tables
    for name, m in [("sat_uniform_6x9", rng.uniform(-1, 1, (6, 9))),
                    ("sat_integer_12x10", rng.integers(0, 1001, (12, 10)).astype(np.float64)),
                    ("sat_fp32_exp_40x1100", rng.exponential(1, (40, 1100)).astype(np.float32).astype(np.float64))]:
        save(name, kind="sat", input=m, table=ref.build_sat(m))

    # CA-CFAR
    def cfar_case(name, m, g, b, pfa, backend="integral"):
        r = ref.cfar2d(m, g, b, pfa, backend)
        save(name, kind="cfar", input=m, params=np.array([g, b, pfa]), backend=backend, mask=r.mask,
             threshold_map=r.threshold_map, det_row=r.detections["row"], det_col=r.detections["col"],
             det_value=r.detections["value"], det_threshold=r.detections["threshold"])

    m = rng.exponential(1.0, (64, 96))
    for (rr, cc) in [(10, 10), (30, 50), (63, 95), (0, 3), (40, 1)]:
        m[rr, cc] += 10 ** 1.5
    cfar_case("cfar_cfg1like_64x96_g2b8", m, 2, 8, 1e-2)
    cfar_case("cfar_cfg1like_64x96_g2b8_naive", m, 2, 8, 1e-2, "naive")
    cfar_case("cfar_integer_48x48_g4b8", rng.integers(0, 501, (48, 48)).astype(np.float64), 4, 8, 1e-3)
    cfar_case("cfar_exp_33x70_g1b3_pfa05", rng.exponential(1.0, (33, 70)), 1, 3, 0.05)
    cfar_case("cfar_tiny_1x2_tie", np.full((1, 2), 5.0), 0, 1, 0.5)

    # spectra (FFTW contract via the oracle provider)
    d = rng.uniform(-1, 1, (3, 50))
    save("spectrum_3x50_L64", kind="spectrum", input=d, fft_length=64, power=ref.slow_time_spectrum(d, 64)[0])
    d = rng.uniform(-1, 1, (2, 600))
    save("spectrum_2x600_L1024", kind="spectrum", input=d, fft_length=1024,
         power=ref.slow_time_spectrum(d, 1024)[0])
    save("spectrum_2x600_L600", kind="spectrum", input=d, fft_length=600,
         power=ref.slow_time_spectrum(d, 600)[0])

    # detect() on a small cfg2-like record (fp32-quantised raw samples)
    m_, n_, prf = 128, 256, 20.0
    mm = np.arange(m_)[:, None]
    t = np.arange(n_)[None, :] / prf
    rec = (rng.uniform(-1, 1, n_)[None, :] + rng.uniform(-1e-3, 1e-3, n_)[None, :] * mm
           + rng.normal(0, 0.1, (m_, n_))
           + 0.5 * np.sin(2 * np.pi * 0.4 * t + 0.3) * np.exp(-((mm - 50.0) ** 2) / 18.0))
    rec = rec.astype(np.float32).astype(np.float64)
    out = ref.detect(rec, prf=prf, guard_radius=1, background_radius=4, pfa=1e-3)
    save("detect_cfg2like_128x256", kind="detect", input=rec, prf=prf, guard=1, train=4, pfa=1e-3,
         band_power=out["band_power"], mask=out["result"].mask, threshold_map=out["result"].threshold_map,
         det_row=out["result"].detections["row"], det_col=out["result"].detections["col"])
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
