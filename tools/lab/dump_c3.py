"""Dump C3's physical SpMV layout (part 0 of 1, f32) for spmv_lab.cu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import synthgen as S
import paper_2201_07498_b200 as T
out = sys.argv[1] if len(sys.argv) > 1 else "/tmp/c3"
os.makedirs(out, exist_ok=True)
A = S.config_matrix("C3")
L = T.plan_layout(A, 1, 0, "f32")
nb = L["nbig"]
# SELL region only: rebase to the start of the SELL storage
z0 = int(L["rowptr"][nb])
L["pcol"][z0:].astype(np.int32).tofile(f"{out}/pcol.bin")
L["pval"][z0:].astype(np.float32).tofile(f"{out}/pval.bin")
sell = L["sell"].copy(); sell[:, 0] -= z0
sell.astype(np.int32).tofile(f"{out}/sell.bin")
L["items"].astype(np.int32).tofile(f"{out}/items.bin")
H = int(min(A.n, 200 * 1024 // 4))
np.array([nb, L["nnonempty"], A.n, H], np.int64).tofile(f"{out}/meta.bin")
bc, bv = L["pcol"][:z0].copy(), L["pval"][:z0].copy()
if os.environ.get("SORT_ROWS") == "1":  # entries of each big row sorted by device column (position)
    rp = L["rowptr"]
    for p in range(nb):
        a, b = rp[p], rp[p + 1]
        o = np.argsort(bc[a:b], kind="stable")
        bc[a:b], bv[a:b] = bc[a:b][o], bv[a:b][o]
bc.astype(np.int32).tofile(f"{out}/bcol.bin")
bv.astype(np.float32).tofile(f"{out}/bval.bin")
L["chunks"].astype(np.int32).tofile(f"{out}/chunks.bin")
print("sell nnz slots", len(L["pcol"]) - z0, "big nnz", z0, "nbig", nb, "pad frac",
      (len(L["pcol"]) - z0) / max(1, (L["rowptr"][L["nnonempty"]] - z0)) - 1)
