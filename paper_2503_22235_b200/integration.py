"""The plugin seam into the reference package (`gridcast`): rebinding its by-name imports to the B200 path.

The reference has no plugin registry or FFI; its modules bind the hot-path functions by name at import
(SURVEY.md §8b): `gridcast.model` imports `natten_block` from `.attention` (model.py:23), `gridcast.rollout`
imports `encode / process / decode` from `.model` (rollout.py:18-27), `gridcast.cli` keeps its own copies of
those plus `blend_latents` and `rollout` (cli.py:32-43).  `install(gridcast)` rebinds every inference caller's
copy in one place (INTEGRATION.md §2 shows the same assignments); `uninstall` restores the originals.

Latents and decoded fields produced by the B200 functions are device-backed (`.values` = float64 numpy); a
reference function that receives one must therefore itself be rebound, which is why the model-level names
are rebound in `gridcast.model` too.  With `operator=True` the operator seam `gridcast.model.natten_block` /
`gridcast.attention.natten_block` is also rebound, so the reference's own model functions still held by
other modules (`gridcast.training`, `gridcast.verify`) call the B200 block — on reference Tensors it returns
reference Tensors, and a call the reference would record on its tape is recorded with the B200 block VJP
(backward.block_vjp) as its backward rule.
"""

from __future__ import annotations

_SAVED: dict = {}

# (module, name) pairs rebound by install(); the value is the attribute of this package that replaces it
_MODEL_LEVEL = {
    "model": ("encode", "process", "decode", "blend_latents"),
    "rollout": ("encode", "process", "decode", "rollout", "forecast"),
    "cli": ("encode", "process", "decode", "blend_latents", "rollout"),
}
_OPERATOR = {"model": ("natten_block",), "attention": ("natten_block",)}


def _replacement(name: str):
    from . import attention, model, rollout
    for mod in (rollout, model, attention):
        if hasattr(mod, name):
            return getattr(mod, name)
    raise AttributeError(name)


def install(gridcast, operator: bool = False, model_level: bool = True) -> None:
    """Rebind the reference's inference entry points (model_level) and / or its natten_block seam (operator)
    to the B200 path.  Idempotent; `uninstall(gridcast)` restores."""
    import importlib
    table = dict(_MODEL_LEVEL) if model_level else {}
    if operator:
        for k, v in _OPERATOR.items():
            table[k] = table.get(k, ()) + v
    for modname, names in table.items():
        mod = importlib.import_module(f"{gridcast.__name__}.{modname}")
        for name in names:
            key = (mod.__name__, name)
            if key not in _SAVED:
                _SAVED[key] = (mod, getattr(mod, name))
            setattr(mod, name, _replacement(name))


def uninstall(gridcast=None) -> None:
    """Restore every name install() rebound."""
    for (_, name), (mod, orig) in list(_SAVED.items()):
        setattr(mod, name, orig)
    _SAVED.clear()


def installed() -> list[str]:
    return sorted(f"{m}.{n}" for m, n in _SAVED)
