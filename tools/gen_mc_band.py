"""Write tests/golden/mc_band.json: the oracle's seeded Monte-Carlo bias/spread band.

The paper gives no bias formula, so the per-overlap mean and sd
of the IP estimation error at psi=100, N=1224 are committed as a regression
band from the oracle's first seeded run. Calls only oracle/ (never the CUDA path).
    python tools/gen_mc_band.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tools.mc_pairs import ensemble  # noqa: E402

M, N, PAIRS, SEED = 100, 1224, 1000, 12345


def main():
    band = {"source": "tools/gen_mc_band.py (oracle only); psi=|a|=|b|=100, N=1224, 1000 maps per overlap",
            "m": M, "N": N, "pairs": PAIRS, "seed": SEED, "overlaps": {}}
    for o in (0, 25, 50, 75, 100):
        E = ensemble(M, o, N, PAIRS, SEED + 100_000 * o)
        err = E[:, 5] - o
        band["overlaps"][str(o)] = {"mean_err": float(err.mean()), "sd_err": float(err.std()),
                                    "max_abs_err": float(abs(err).max())}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "tests", "golden", "mc_band.json")
    with open(path, "w") as f:
        json.dump(band, f, indent=1)
    print(json.dumps(band, indent=1))


if __name__ == "__main__":
    main()
