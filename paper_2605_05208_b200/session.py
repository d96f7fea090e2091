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


def session_for(inst, consts=None, nbr=None, device: int = 0) -> Session:
    """Session keyed by the identity of the instance and neighbour lists."""
    key = (id(inst), id(nbr) if nbr is not None else None, device)
    s = _SESSIONS.get(key)
    if s is not None and s.inst is inst and s.nbr is nbr:
        if consts is None or (consts.gamma, consts.theta) == (s.consts.gamma, s.consts.theta):
            return s
    if consts is None:
        consts = ScalingConstants.from_instance(inst)
    s = Session(inst, consts, nbr, device)
    _SESSIONS[key] = s
    try:
        weakref.finalize(inst, _SESSIONS.pop, key, None)
    except TypeError:
        pass
    return s
