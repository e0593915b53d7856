"""Shared scenario builders (reference JSON schema, proj/README.md:77-113)."""
import copy
import json
import os

SLAB_MATERIALS = {  # proj/configs/slab_nonlinear_rkc_spe.json:22-47
    "1": {"eps_r": 3.0, "conductivity": {"kind": "constant", "kappa": 1e-9}},
    "2": {"eps_r": 12.0, "conductivity": {"kind": "microvaristor", "kappa_lo": 1e-10, "kappa_hi": 3e-6,
                                          "e_switch": 5e5, "width": 5e4}},
    "3": {"eps_r": 3.0, "conductivity": {"kind": "constant", "kappa": 1e-9}},
}


def cube(n, jitter=0.0, order=1, estimator="spe", precond="amg", amplitude=4e4 / 0.012, planes=(1 / 3, 2 / 3),
         materials=None):
    """Unit cube with three layers; hv amplitude scaled so fields match the
    reference nonlinear slab."""
    return {
        "name": f"cube{n}",
        "mesh": {"box": {"nx": n, "ny": n, "nz": n, "lx": 1.0, "ly": 1.0, "lz": 1.0,
                         "z_planes": list(planes), "regions": [1, 2, 3], "jitter": jitter}},
        "order": order,
        "materials": copy.deepcopy(materials or SLAB_MATERIALS),
        "excitations": {"hv": {"kind": "sinusoid", "amplitude": amplitude, "frequency": 50.0},
                        "ground": {"kind": "constant", "value": 0.0}},
        "integrator": {"kind": "rkc", "tolerance": 1e-2, "t_end": 0.02, "dt0": 1e-5},
        "solver": {"preconditioner": precond, "rel_tol": 1e-12, "max_iter": 500},
        "estimator": {"mode": estimator, "window": 8},
    }


def matfree_setup(order, nonlinear, n=3):
    """proj/tests/test_matfree.cpp:22-38 (unit box, layers at 0.5)."""
    mats = {"1": {"eps_r": 2.0, "conductivity": {"kind": "constant", "kappa": 1e-8}},
            "2": {"eps_r": 5.0, "conductivity": ({"kind": "microvaristor", "kappa_lo": 1e-10, "kappa_hi": 1e-4,
                                                   "e_switch": 0.5, "width": 0.2} if nonlinear else
                                                  {"kind": "constant", "kappa": 3e-9})}}
    return {"mesh": {"box": {"nx": n, "ny": n, "nz": n, "lx": 1, "ly": 1, "lz": 1, "z_planes": [0.5],
                             "regions": [1, 2]}},
            "order": order, "materials": mats,
            "excitations": {"ground": {"kind": "constant", "value": 0.0},
                            "hv": {"kind": "constant", "value": 1.0}}}


# verbatim copies of proj/configs/*.json (tests/golden/make_reference_configs.py):
# /root/reference does not exist on the GPU box
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_configs.json")) as _f:
    REFERENCE_CONFIGS = json.load(_f)


def slab_reference(name):
    return copy.deepcopy(REFERENCE_CONFIGS[name])


TINY_SLAB = {  # proj/tests/test_scenario.cpp:21-39 (tiny_slab_json)
    "name": "tiny",
    "mesh": {"box": {"nx": 3, "ny": 3, "nz": 6, "lx": 0.01, "ly": 0.01, "lz": 0.02, "z_planes": [0.01],
                     "regions": [1, 2]}},
    "order": 1,
    "materials": {"1": {"eps_r": 2.0, "conductivity": {"kind": "constant", "kappa": 1e-8}},
                  "2": {"eps_r": 5.0, "conductivity": {"kind": "constant", "kappa": 5e-9}}},
    "excitations": {"ground": {"kind": "constant", "value": 0.0},
                    "hv": {"kind": "sinusoid", "amplitude": 100.0, "frequency": 50.0}},
    "integrator": {"kind": "rkc", "tolerance": 1e-2, "t_end": 2e-3, "dt0": 1e-5},
    "solver": {"preconditioner": "amg", "rel_tol": 1e-12, "max_iter": 500},
    "estimator": {"mode": "spe", "window": 8},
    "probes": [[0.005, 0.005, 0.01]],
    "output": {"metrics_csv": "", "probe_csv": "", "solves_csv": ""},
}


def tiny_slab(**over):
    c = copy.deepcopy(TINY_SLAB)
    for k, v in over.items():
        c[k] = v
    return c
