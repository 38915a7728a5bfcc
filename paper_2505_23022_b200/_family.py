"""Resolve the caller's type family (this package's or the reference's ``slosim``).

The drop-in functions accept objects of either package: a ``slosim.SimConfig``
with ``slosim`` ``Request``s, or this package's own mirrors.  They read plain
fields only, and build their results (``RequestOutcome`` with the caller's
``Status`` members, ``RunningEntry``, ``StepPlan``, ``AdmissionRecord``,
``EventLog`` / ``StepRecord``) from the caller's own classes, so identity checks
such as ``o.status is Status.COMPLETED`` in the reference's ``summarize``
(``report.py:71-127``) hold.
"""

from __future__ import annotations

import importlib
import sys
from types import SimpleNamespace

_OWN = __name__.rsplit(".", 1)[0]
_cache: dict[str, SimpleNamespace] = {}


def _load(root: str) -> SimpleNamespace:
    def mod(name):
        full = f"{root}.{name}"
        m = sys.modules.get(full)
        return m if m is not None else importlib.import_module(full)

    core, st = mod("core"), mod("schedtypes")
    ns = SimpleNamespace(
        root=root, Status=core.Status, RequestOutcome=core.RequestOutcome,
        WaitingItem=st.WaitingItem, RunningEntry=st.RunningEntry, StepPlan=st.StepPlan,
        AdmissionRecord=st.AdmissionRecord, SchedulerState=st.SchedulerState)
    sim = sys.modules.get(f"{root}.simengine")
    if sim is None and root == _OWN:
        sim = mod("simengine")
    if sim is not None:
        ns.EventLog, ns.StepRecord = sim.EventLog, sim.StepRecord
    return ns


def family(*objs) -> SimpleNamespace:
    """The type family of the first object that belongs to a known package
    (``slosim`` or this one); this package's own when none does."""
    root = _OWN
    for o in objs:
        if o is None:
            continue
        r = type(o).__module__.split(".", 1)[0]
        if r != "builtins":
            root = r
            break
    ns = _cache.get(root)
    if ns is None:
        try:
            ns = _load(root)
        except (ImportError, AttributeError):
            ns = _load(_OWN)
        _cache[root] = ns
    if not hasattr(ns, "EventLog"):  # simengine imported after the first lookup
        ns = _cache[root] = _load(root)
    return ns


def status_code(status) -> int:
    """C ABI code (0..3) of either package's ``Status`` member (by value)."""
    return {"completed": 0, "rejected_ttft": 1, "rejected_admission": 2,
            "incomplete": 3}[status.value]
