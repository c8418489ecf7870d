python - <<'PY'
import torch
from cuda.bindings import runtime as rt
for a in ["cudaDevAttrL2CacheSize","cudaDevAttrMaxPersistingL2CacheSize","cudaDevAttrMaxAccessPolicyWindowSize"]:
    print(a, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0))
PY
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1; }
for c in c2s18 c2s20 c2 c2s24; do echo "$(run $c)"; done
for h in 0.25 1.0; do echo "c2 hot=$h $(PRGPU_HOT_FRAC=$h run c2)"; done
