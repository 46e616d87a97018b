"""Host model of one slab rank for the CPU (gloo) multi-process tests: the C oracle steps the
rank's stored tiles (layout and local tables from the native splbm_slab_layout — the same code the
device engine uses), numpy packs/unpacks the face layers with the device halo kernel's slot
formula, and paper_1703_08015_b200.slab.HaloExchange moves them over torch.distributed."""
import numpy as np

import paper_1703_08015_b200 as P
from paper_1703_08015_b200 import slab


def face_dirs(d):
    lat = P.solver_lattice(d)
    ax = 2 if d == 3 else 1
    ups = [i for i in range(lat.q) if lat.e[i][ax] == 1]
    downs = [i for i in range(lat.q) if lat.e[i][ax] == -1]
    return ups, downs


class HostSlabRank:
    """single_copy=True: one PDF array stepped with the AA ordering (oracle_aa_step, owned tiles
    only); before a phase-1 step the owners' natural-state faces go to the neighbours' halos
    (pack/unpack), after it the halo face slots the scatter wrote go back to their owners
    (pack_back/unpack_back) — the schedule of SlabRun's torch transport in single-copy mode."""

    def __init__(self, O, g, a, tau, per, z0, z1, inc=False, single_copy=False):
        self.O, self.g, self.a = O, g, a
        self.d = g.d
        self.q = 9 if g.d == 2 else 19
        self.n_tn = a * a * (a if g.d == 3 else 1)
        self.face = self.n_tn // a
        self.lay = slab.slab_layout(g, a, per, z0, z1, tables=True)
        L = self.lay
        self.S = L["n_low"] + L["n_own"] + L["n_high"]
        tl = L["types_local"]
        self.ttypes = np.ascontiguousarray(tl & 3)
        self.bcdeg = np.ascontiguousarray((tl >> 2) & 1)
        self.nb = np.ascontiguousarray(L["nb_local"])
        tg = P.build_tile_grid(g, a, per, with_neighbours=False)
        gid = np.concatenate([L["g_low0"] + np.arange(L["n_low"]), L["g_own0"] + np.arange(L["n_own"]),
                              L["g_high0"] + np.arange(L["n_high"])]).astype(np.int64)
        self.gid = gid
        x, y, z = O.tile_node_coords(tg.origins[gid], a, g.d)
        n = self.S * self.q * self.n_tn
        self.pdf = [np.zeros(max(n, 1)), np.zeros(max(n, 1))]
        rho, ux, uy, uz = O.wavy(x, y, z)
        O.lib().oracle_t2c_initialize(g.d, self.S, self.n_tn, int(inc), rho, ux, uy, uz,
                                      self.pdf[0], self.pdf[1])
        self.read = 0
        self.single_copy = single_copy
        self.state = 0  # single copy: 0 natural layout, 1 swapped
        self.inv_tau = 1.0 / tau
        self.inc = int(inc)
        self.ups, self.downs = face_dirs(g.d)

    def step(self):
        if self.single_copy:
            L = self.lay
            ok = self.O.lib().oracle_aa_step(self.d, self.a, L["n_low"], L["n_low"] + L["n_own"],
                                             self.ttypes, self.nb, self.bcdeg, self.pdf[0],
                                             1 + self.state, self.inv_tau, self.inc,
                                             np.asarray(self.g.bc.velocity, np.float64),
                                             self.g.bc.density)
            self.state ^= 1
            return ok
        ok = self.O.lib().oracle_t2c_step(self.d, self.a, self.S, self.ttypes, self.nb, self.bcdeg,
                                          self.pdf[self.read], self.pdf[1 - self.read], self.inv_tau,
                                          self.inc, np.asarray(self.g.bc.velocity, np.float64),
                                          self.g.bc.density, 1, None)
        self.read = 1 - self.read
        return ok

    def _slots(self, tile0, ntiles, layer, dirs):
        t = tile0 + np.arange(ntiles)[:, None, None]
        j = np.asarray(dirs)[None, :, None]
        f = np.arange(self.face)[None, None, :]
        return (((t * self.q + j) * self.n_tn) + layer * self.face + f).ravel()

    def pack(self, lo, hi):
        L = self.lay
        cur = self.pdf[self.read]
        if lo.numel():
            lo.numpy()[:] = cur[self._slots(L["n_low"], L["send_low_tiles"], 0, self.downs)]
        if hi.numel():
            hi.numpy()[:] = cur[self._slots(L["n_low"] + L["n_own"] - L["send_high_tiles"],
                                            L["send_high_tiles"], self.a - 1, self.ups)]

    def unpack(self, lo, hi):
        L = self.lay
        cur = self.pdf[self.read]
        if lo is not None and lo.numel():
            cur[self._slots(0, L["n_low"], self.a - 1, self.ups)] = lo.numpy()
        if hi is not None and hi.numel():
            cur[self._slots(L["n_low"] + L["n_own"], L["n_high"], 0, self.downs)] = hi.numpy()

    def pack_back(self, lo, hi):
        """Single copy, after a phase-1 step: the halo face slots my scatter wrote (low halo top
        layer, upward dirs; high halo bottom layer, downward dirs) go back to their owners."""
        L = self.lay
        cur = self.pdf[0]
        if lo.numel():
            lo.numpy()[:] = cur[self._slots(0, L["n_low"], self.a - 1, self.ups)]
        if hi.numel():
            hi.numpy()[:] = cur[self._slots(L["n_low"] + L["n_own"], L["n_high"], 0, self.downs)]

    def _written_by_neighbour(self, tile0, ntiles, layer, dirs):
        """Per slot (x, k) of an owned face: did the neighbour's phase-1 scatter write it? Only
        when the downstream node x + e_k exists and is non-solid (its gather of k from x is not
        blocked); otherwise x's own bounce-back owns the slot and it must not be overwritten."""
        lat = P.solver_lattice(self.d)
        a, d = self.a, self.d
        out = np.zeros((ntiles, len(dirs), self.face), bool)
        for ti in range(ntiles):
            t = tile0 + ti
            for jn, k in enumerate(dirs):
                e = lat.e[k]
                for f in range(self.face):
                    p = layer * self.face + f
                    l = [p % a, (p // a) % a, p // (a * a)] if d == 3 else [p % a, p // a, 0]
                    dc = [0, 0, 0]
                    for c in range(d):
                        l[c] += e[c]
                        if l[c] < 0:
                            dc[c], l[c] = -1, l[c] + a
                        elif l[c] >= a:
                            dc[c], l[c] = 1, l[c] - a
                    s = self.nb[t * 27 + (dc[0] + 1) + 3 * ((dc[1] + 1) + 3 * (dc[2] + 1))]
                    if s != 0xFFFFFFFF:
                        out[ti, jn, f] = self.ttypes[s * self.n_tn + l[0] + a * (l[1] + a * l[2])] != 0
        return out.ravel()

    def unpack_back(self, lo, hi):
        L = self.lay
        cur = self.pdf[0]
        if lo is not None and lo.numel():
            args = (L["n_low"], L["send_low_tiles"], 0, self.downs)
            m = self._written_by_neighbour(*args)
            cur[self._slots(*args)[m]] = lo.numpy()[m]
        if hi is not None and hi.numel():
            args = (L["n_low"] + L["n_own"] - L["send_high_tiles"], L["send_high_tiles"], self.a - 1,
                    self.ups)
            m = self._written_by_neighbour(*args)
            cur[self._slots(*args)[m]] = hi.numpy()[m]

    def sizes_back(self):
        f = self.sizes()
        return {"send_low": f["recv_low"], "send_high": f["recv_high"], "recv_low": f["send_low"],
                "recv_high": f["send_high"]}

    def sizes(self):
        L = self.lay
        per_tile = len(self.ups) * self.face * 8
        return {"send_low": L["send_low_tiles"] * per_tile, "send_high": L["send_high_tiles"] * per_tile,
                "recv_low": L["n_low"] * per_tile, "recv_high": L["n_high"] * per_tile}

    def owned_pdf(self):
        L = self.lay
        st = self.q * self.n_tn
        return self.pdf[self.read][L["n_low"] * st:(L["n_low"] + L["n_own"]) * st]
