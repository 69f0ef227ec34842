"""The PBMC-scale sparse/COCA spectrum stage of bench.py alone (both Gram back ends):
python tools/pbmc_probe.py  (GGM_GRAM_TC=0/1 selects fp64 DSYRK / the tensor-core Gram)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_19892_b200 as G  # noqa: E402

print(json.dumps({"GGM_GRAM_TC": os.environ.get("GGM_GRAM_TC"),
                  **bench.sparse_spectrum_timing(G, torch)}), flush=True)
