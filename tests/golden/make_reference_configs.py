"""Regenerate tests/golden/reference_configs.json from the reference's committed
scenario configs (proj/configs/*.json). Run in the build container, where
/root/reference exists; the GPU box only reads the committed JSON."""
import json
import os

SRC = "/root/reference/proj/configs"
NAMES = ["smoke", "slab_nonlinear_rkc_spe", "slab_linear_rkc", "slab_linear_rkc_previous", "slab_linear_rkc_spe",
         "slab_order2_rkc", "slab_linear_euler", "slab_nonlinear_rkc_pod_fixed", "slab_nonlinear_rkc_pod_rolling",
         "slab_nonlinear_sdirk"]

if __name__ == "__main__":
    out = {n: json.load(open(os.path.join(SRC, n + ".json"))) for n in NAMES}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_configs.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path)
