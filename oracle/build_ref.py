"""Build the reference's own compiled tile kernel into oracle/_ref/ (TEST /
BASELINE INFRASTRUCTURE ONLY — never on the product path).

The reference's `compiled` backend is one Cython file,
/root/reference/pkg/src/omniattn/_kernels/_core.pyx (masked_block_attention,
_core.pyx:14-101). This recipe cythonizes it IN PLACE OF the reference's own
setup.py (pkg/setup.py:12-33: language_level 3, boundscheck/wraparound off,
cdivision on, -O3, the NumPy 1.7 API macro) with every output under
oracle/_ref/ (git-ignored, shipped to the GPU box with the snapshot). The
reference source is read where it lies and never copied into the repo.

    python -m oracle.build_ref        (or oracle.build_ref.build())

`load_core()` imports the built module. Its only import-time dependency on the
reference package is `omniattn.errors.ConsistencyError` (_core.pyx:9); when
the reference package is not importable (the GPU box) a stand-in exception
class of that name is registered for it, so the kernel runs unchanged.
"""

import importlib.util
import pathlib
import subprocess
import sys
import sysconfig
import types

HERE = pathlib.Path(__file__).resolve().parent
REF_PYX = pathlib.Path("/root/reference/pkg/src/omniattn/_kernels/_core.pyx")
OUT_DIR = HERE / "_ref"
C_FILE = OUT_DIR / "_core.c"
SO_FILE = OUT_DIR / ("_core" + sysconfig.get_config_var("EXT_SUFFIX"))


def available():
    return SO_FILE.exists()


def build(force=False):
    """Compile the reference kernel; a no-op when the reference tree is absent
    (the GPU box ships the prebuilt .so) or the build is current."""
    if not REF_PYX.exists():
        return SO_FILE if SO_FILE.exists() else None
    if not force and SO_FILE.exists() and SO_FILE.stat().st_mtime >= REF_PYX.stat().st_mtime:
        return SO_FILE
    import numpy as np

    OUT_DIR.mkdir(exist_ok=True)
    subprocess.run([sys.executable, "-m", "cython", "-3",
                    "--directive", "boundscheck=False,wraparound=False,cdivision=True",
                    "--module-name", "omniattn._kernels._core",
                    "-o", str(C_FILE), str(REF_PYX)], check=True)
    subprocess.run(["gcc", "-O3", "-shared", "-fPIC", "-fwrapv",
                    "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION",
                    "-I", sysconfig.get_paths()["include"], "-I", np.get_include(),
                    "-o", str(SO_FILE), str(C_FILE)], check=True)
    return SO_FILE


_core = None


def load_core():
    """The reference's compiled masked_block_attention module (NAME == "compiled")."""
    global _core
    if _core is not None:
        return _core
    if not SO_FILE.exists():
        raise ImportError(f"reference kernel not built ({SO_FILE}); run python -m oracle.build_ref")
    try:
        import omniattn.errors  # noqa: F401  (the real reference, when importable)
    except ImportError:
        if "omniattn.errors" not in sys.modules:
            pkg = sys.modules.setdefault("omniattn", types.ModuleType("omniattn"))
            pkg.__path__ = []
            err = types.ModuleType("omniattn.errors")

            class ConsistencyError(Exception):
                """Stand-in for omniattn.errors.ConsistencyError (errors.py)."""

            err.ConsistencyError = ConsistencyError
            sys.modules["omniattn.errors"] = err
            pkg.errors = err
    spec = importlib.util.spec_from_file_location("omniattn._kernels._core", SO_FILE)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    _core = mod
    return mod


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
