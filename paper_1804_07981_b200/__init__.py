"""B200-native Biham-Middleton-Levine traffic CA — drop-in for the reference `bml` package.

Same public surface as the reference (/root/reference/proj/python/bml/__init__.py,
bindings/py_module.cpp:38-158): ``init_grid``, ``step``, ``simulate``, ``Grid``,
``count_vehicles``, ``classify``, ``StepMetrics`` ... with ``Backend.b200`` as the
default engine. Stepping runs only on the GPU through ``libbml_dev.so``
(include/bml_dev.h); importing fails loudly if the native extension is missing —
there is no CPU fallback.

    import paper_1804_07981_b200 as bml
    grid = bml.init_grid(n=1024, rho=0.38, seed=1)
    final, metrics = bml.simulate(grid, 4096)
"""
import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))

try:
    from ._bml import (  # noqa: F401
        Backend,
        Cell,
        DeviceLattice,
        Grid,
        Phase,
        Regime,
        StepMetrics,
        VerifyReport,
        __version__,
        backend_from_name,
        classify,
        count_vehicles,
        device_count,
        encode_ppm,
        init_grid,
        lane_width,
        library_version,
        moved_in_phase,
        simulate,
        step,
        step_phase,
        vehicles_per_species,
        verify_backends,
        verify_device,
        write_ppm,
    )
except ImportError as exc:  # pragma: no cover - exercised only on broken installs
    raise ImportError(
        "paper_1804_07981_b200: native extension not built or not loadable "
        f"({exc}); run `python -c 'import __graft_entry__ as g; g.build()'` first"
    ) from exc

LIB_DEV = _os.path.join(_HERE, "libbml_dev.so")

__all__ = [
    "Backend",
    "Cell",
    "DeviceLattice",
    "Grid",
    "Phase",
    "Regime",
    "StepMetrics",
    "VerifyReport",
    "__version__",
    "backend_from_name",
    "classify",
    "count_vehicles",
    "device_count",
    "encode_ppm",
    "init_grid",
    "lane_width",
    "library_version",
    "moved_in_phase",
    "simulate",
    "step",
    "step_phase",
    "vehicles_per_species",
    "verify_backends",
    "verify_device",
    "write_ppm",
    "LIB_DEV",
]
