"""Write a workloads config graph as a flat binary (int64 n, nnz, off[n+1], int32 cols[nnz])."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import workloads as W  # noqa: E402

g, _, _ = W.load_config(sys.argv[1], with_lambda=False)
with open(sys.argv[2], "wb") as f:
    np.array([g.n, g.nnz], dtype=np.int64).tofile(f)
    g.offsets.astype(np.int64).tofile(f)
    g.cols.astype(np.int32).tofile(f)
