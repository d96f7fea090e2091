"""Per-instance device sessions: one uploaded instance per (instance, lists,
device) and reusable populations, so repeated API calls do not re-upload the
distance matrix."""
from __future__ import annotations

import weakref

from .device import DeviceInstance, Population
from .evaluation import ScalingConstants

_SESSIONS: dict = {}


def _ref(obj):
    """Weak reference where the type allows one: a cache entry must not keep its
    instance alive, or its finalizer (which frees the device copies) never runs."""
    try:
        return weakref.ref(obj)
    except TypeError:
        return lambda: obj


class Session:
    def __init__(self, inst, consts, nbr, device: int):
        self._inst = _ref(inst)
        self.consts = consts
        self.nbr = nbr
        self.device = device
        self.dinst = DeviceInstance(inst, consts, nbr, device)
        self._single = None
        self._single_sig = None

    @property
    def inst(self):
        return self._inst()

    def single(self, sol, lam):
        """A B=1 population holding `sol` (re-uploaded only when it changed)."""
        sig = tuple((r.depart, r.arrive, tuple(r.customers)) for r in sol.routes)
        J, K = Population.caps_for([sol], self.inst)
        p = self._single
        if p is None or p.J_cap < J or p.K_cap < K:
            p = self._single = Population(self.dinst, 1, J, K, 1 << 12)
            self._single_sig = None
        if self._single_sig != sig:
            p.upload([sol], [lam])
            self._single_sig = sig
        return p

    def invalidate(self):
        self._single_sig = None


def same_consts(a, b) -> bool:
    return (a.gamma, a.theta) == (b.gamma, b.theta)


def session_for(inst, consts=None, nbr=None, device: int = 0) -> Session:
    """The device session of an instance on a device.

    One entry per (instance, device, with/without lists): a call with other
    neighbour lists or other scaling constants (baked into the device
    instance) replaces the entry, which frees the old device instance and its
    populations -- repeated runs that build fresh lists do not accumulate
    device memory.  The entry goes with the instance (weak reference)."""
    key = (id(inst), device, nbr is None)
    s = _SESSIONS.get(key)
    if s is not None and s.inst is inst and s.nbr is nbr:
        if consts is None or same_consts(consts, s.consts):
            return s
    if consts is None:
        consts = ScalingConstants.from_instance(inst)
    _SESSIONS.pop(key, None)  # drop the stale entry before allocating the new one
    s = Session(inst, consts, nbr, device)
    _SESSIONS[key] = s
    try:
        weakref.finalize(inst, _SESSIONS.pop, key, None)
    except TypeError:
        pass
    return s
