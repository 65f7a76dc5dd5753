"""Drop the GPU path into an imported reference package (``jfft``).

The reference has no plugin registry: its operator API is the set of
module-level functions re-exported by ``jfft/__init__.py:5-21``, and each
importing module binds them by name at import time.  This
rebinds every binding site so that the reference's own experiments, topology
optimisation, CLI and Newton driver run on libjfftb200:

  preconditioners.{apply_system, make_operator, apply_green, apply_jacobi,
                   apply_jacobi_half, apply_green_jacobi, assemble_green,
                   assemble_jacobi, build_preconditioner, Preconditioner}
  operators.{apply_system, assemble_rhs, total_strain, residual_force,
             homogenized_stress}
  solver.{apply_system, residual_force, apply_green, assemble_green,
          build_preconditioner, pcg}
  experiments.{assemble_rhs, homogenized_stress, assemble_green,
                build_preconditioner, pcg}
  topopt.{assemble_rhs, total_strain, assemble_green, build_preconditioner, pcg}
  microstructures.{gaussian_filter, threshold, rescale_contrast, total_contrast}
      (experiments.py:18 reaches them through the module object)
  grid.{save_field, load_field}, experiments.{save_field, load_field}
  jfft.{...the same names}

``SystemOperator`` objects stay the reference's own (they are plain data);
the device copy of the density is attached to them lazily.  Solver aborts are
raised as the reference's ``SolverAbortError``.
"""

from __future__ import annotations

import importlib

from . import fieldio as _fieldio
from . import generators as _gen
from . import operators as _ops
from . import preconditioners as _pc
from . import solver as _solver

_TARGETS = {
    "preconditioners": ["apply_system", "apply_green", "apply_jacobi", "apply_jacobi_half",
                        "apply_green_jacobi", "assemble_green", "assemble_jacobi",
                        "build_preconditioner", "Preconditioner"],
    "operators": ["apply_system", "assemble_rhs", "total_strain", "residual_force",
                  "homogenized_stress"],
    "solver": ["apply_system", "residual_force", "apply_green", "assemble_green",
               "build_preconditioner", "pcg"],
    "experiments": ["assemble_rhs", "homogenized_stress", "assemble_green",
                    "build_preconditioner", "pcg", "save_field", "load_field"],
    "topopt": ["assemble_rhs", "total_strain", "assemble_green", "build_preconditioner", "pcg"],
    "microstructures": ["gaussian_filter", "threshold", "rescale_contrast", "total_contrast"],
    "grid": ["save_field", "load_field"],
    "": ["apply_system", "assemble_rhs", "total_strain", "residual_force", "homogenized_stress",
         "apply_green", "apply_jacobi", "apply_jacobi_half", "apply_green_jacobi",
         "assemble_green", "assemble_jacobi", "build_preconditioner", "Preconditioner", "pcg"],
}


def _replacement(name: str, ref_solver, original=None):
    if name == "pcg":
        def pcg(op, rhs, preconditioner, green, eta=_solver.DEFAULT_ETA_CG,
                max_iter=_solver.DEFAULT_MAX_ITER):
            return _solver.pcg(op, rhs, preconditioner, green, eta=eta, max_iter=max_iter,
                               abort_error=ref_solver.SolverAbortError)
        pcg.__doc__ = _solver.pcg.__doc__
        return pcg
    if name == "load_field":
        ref_grid = importlib.import_module(ref_solver.__name__.rsplit(".", 1)[0] + ".grid")

        def load_field(basepath):
            return _fieldio.load_field(basepath, module=ref_grid)
        load_field.__doc__ = _fieldio.load_field.__doc__
        return load_field
    if name == "assemble_jacobi" and original is not None:
        ref_pc = importlib.import_module(ref_solver.__name__.rsplit(".", 1)[0] + ".preconditioners")

        def assemble_jacobi(op):
            # The device diagonal runs its d 2^d comb probes inside the library.
            # If the caller has wrapped the module-level ``apply_system`` (the
            # reference's probing loop calls it by that name,
            # preconditioners.py:109-115; its own test counts the calls), the
            # reference's loop runs instead, through the caller's wrapper --
            # the same probes, each applied on the device, the same diagonal.
            if getattr(ref_pc, "apply_system", None) is not _ops.apply_system:
                return original(op)
            return _pc.assemble_jacobi(op)
        assemble_jacobi.__doc__ = _pc.assemble_jacobi.__doc__
        return assemble_jacobi
    for mod in (_ops, _pc, _solver, _gen, _fieldio):
        if hasattr(mod, name):
            return getattr(mod, name)
    raise AttributeError(name)


def _child_plug(package: str) -> None:
    """Initializer of the sweep pool's worker processes."""
    plug_into_reference(package)


def _pool_factory(package: str, original):
    """The reference's parameter sweeps fan out over a fork-based
    ``ProcessPoolExecutor`` (experiments.py:326-330).  A process that has
    already used CUDA cannot fork workers that use it, so the plugged-in
    sweep starts its workers with ``spawn`` and plugs the GPU path into each
    of them (the cells then run on libjfftb200 as well)."""
    import functools
    import multiprocessing as mp

    @functools.wraps(original)
    def make(*args, **kwargs):
        kwargs.setdefault("mp_context", mp.get_context("spawn"))
        kwargs.setdefault("initializer", _child_plug)
        kwargs.setdefault("initargs", (package,))
        return original(*args, **kwargs)
    return make


def plug_into_reference(package: str = "jfft") -> dict:
    """Rebind the reference's binding sites; returns the originals so that
    :func:`unplug` can restore them."""
    ref_solver = importlib.import_module(f"{package}.solver")
    saved = {}
    try:
        exp = importlib.import_module(f"{package}.experiments")
    except ImportError:
        exp = None
    if exp is not None and hasattr(exp, "ProcessPoolExecutor") and \
            not getattr(exp.ProcessPoolExecutor, "_jfftb_spawn", False):
        saved[(exp.__name__, "ProcessPoolExecutor")] = exp.ProcessPoolExecutor
        factory = _pool_factory(package, exp.ProcessPoolExecutor)
        factory._jfftb_spawn = True
        exp.ProcessPoolExecutor = factory
    for modname, names in _TARGETS.items():
        full = package if modname == "" else f"{package}.{modname}"
        try:
            mod = importlib.import_module(full)
        except ImportError:
            continue
        for name in names:
            if hasattr(mod, name):
                saved[(full, name)] = getattr(mod, name)
                setattr(mod, name, _replacement(name, ref_solver, original=saved[(full, name)]))
    return saved


def unplug(saved: dict) -> None:
    for (full, name), obj in saved.items():
        setattr(importlib.import_module(full), name, obj)
