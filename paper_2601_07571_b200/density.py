"""Density-map generation on the B200 (drop-in for the reference's
density.py: GenerationConfig :44-71, DensityMap :74-91, Timings :94-103,
accumulate_fixation :136-200, generate :203-227, normalize :230-244).

`generate` uploads the scene once into a `ScenePlan` (occluder triangles and
sample positions resident in HBM), streams the fixation table through the
extension in batches (host setup of batch i+1 overlaps the GPU work of batch
i) and reads the per-sample values back.  Per-sample accumulation order is the
fixation log order, so results are deterministic run to run.
"""

from __future__ import annotations

import atexit
import ctypes
import os
import math
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigError
from .gaze import DEFAULT_THETA, GazeCone, fixation_table

__all__ = ["GenerationConfig", "DensityMap", "Timings", "ScenePlan", "accumulate_fixation", "generate",
           "normalize", "DEFAULT_K", "DEFAULT_EPS_ABS", "DEFAULT_EPS_REL", "DEFAULT_RESOLUTION"]

DEFAULT_K = 40000.0
DEFAULT_EPS_ABS = 1e-3
DEFAULT_EPS_REL = 1e-3
DEFAULT_RESOLUTION = 512


@dataclass
class GenerationConfig:
    k: float = DEFAULT_K
    theta: float = DEFAULT_THETA
    zbuffer_resolution: int = DEFAULT_RESOLUTION
    epsilon_abs: float = DEFAULT_EPS_ABS
    epsilon_rel: float = DEFAULT_EPS_REL
    time_window: tuple | None = None
    filtering_enabled: bool = True
    object_include_list: set | None = None

    def validate(self) -> "GenerationConfig":
        if self.k <= 0:
            raise ConfigError(f"k must be > 0, got {self.k}")
        if not 0 < self.theta < math.pi / 2:
            raise ConfigError(f"theta must be in (0, pi/2), got {self.theta}")
        if self.zbuffer_resolution < 1:
            raise ConfigError(f"zbuffer_resolution must be >= 1, got {self.zbuffer_resolution}")
        if self.epsilon_abs < 0 or self.epsilon_rel < 0:
            raise ConfigError("epsilon values must be >= 0")
        if self.time_window is not None and self.time_window[0] > self.time_window[1]:
            raise ConfigError(f"empty time window {self.time_window}")
        return self

    def cone(self) -> GazeCone:
        return GazeCone.from_theta(self.theta)


@dataclass
class DensityMap:
    """Per-object value arrays + tracked global max (reference density.py:74-91).

    A map fed by accumulate_fixation may hold its newest values on the GPU
    only (see _DeviceLink): reading `.values` brings them back first, into the
    same arrays, so the map always looks like the reference's."""

    values: dict
    global_max: float = 0.0
    normalized: bool = False

    def __getattribute__(self, name):
        if name == "values" or name == "global_max":
            d = object.__getattribute__(self, "__dict__")
            link = d.get("_device_link")
            if link is not None:
                link.expose(self) if name == "values" else link.flush()
            if name == "values":
                d.pop("_zero", None)
        return object.__getattribute__(self, name)

    def __setattr__(self, name, value):
        if name == "values" or name == "global_max":
            link = self.__dict__.get("_device_link")
            if link is not None:  # a caller overwriting the map: settle the queued fixations first
                link.expose(self)
            if name == "values":
                self.__dict__.pop("_zero", None)
        object.__setattr__(self, name, value)

    @classmethod
    def zeros(cls, sampled_meshes: dict) -> "DensityMap":
        dm = cls({oid: np.zeros(sm.total_samples) for oid, sm in sampled_meshes.items()})
        dm.__dict__["_zero"] = True  # known all-zero until handed out: accumulate_fixation clears the
        return dm                    # device accumulator instead of uploading zeros

    @property
    def total_samples(self) -> int:
        return sum(len(v) for v in self.values.values())

    def copy(self) -> "DensityMap":
        return DensityMap({k: v.copy() for k, v in self.values.items()}, self.global_max, self.normalized)


@dataclass
class Timings:
    """Seconds per phase.  cull = occluder cone cull + clip + projection
    (device), rasterize = screen binning + evaluation of the z-buffer texels
    the depth test reads (device), accumulate = NDC filter + cone + depth test
    + Gaussian (device, both sample passes), setup = host fixation setup."""

    phases: dict = field(default_factory=lambda: {"cull": 0.0, "rasterize": 0.0, "accumulate": 0.0,
                                                  "normalize": 0.0})

    def add(self, phase: str, seconds: float) -> None:
        self.phases[phase] = self.phases.get(phase, 0.0) + seconds


def _included_ids(scene, config) -> list:
    ids = [o.object_id for o in scene.objects]
    if config.object_include_list is None:
        return ids
    return [oid for oid in ids if oid in config.object_include_list]


class ScenePlan:
    """A scene resident on one GPU: all objects' world triangles (occluders)
    and the included objects' world sample positions + value slots."""

    def __init__(self, scene, sampled_meshes: dict, included: list, device: int = 0):
        lib = _native.load()
        self.device = device
        self.scene = scene
        self.sampled_meshes = sampled_meshes
        h = ctypes.c_void_p()
        _native.check(lib.gm_plan_create(device, ctypes.byref(h)), "gm_plan_create")
        self._h = h
        self._lib = lib
        # one process per GPU (torchrun): split the host cores between the local ranks so
        # their fixation-setup thread pools do not oversubscribe the node
        local = int(os.environ.get("LOCAL_WORLD_SIZE", "1") or 1)
        if local > 1:
            cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
            _native.check(lib.gm_plan_set_host_threads(h, max(1, cores // local)), "gm_plan_set_host_threads")
        objs = list(scene.objects)
        inc = set(included)
        tri_counts, tris, xforms, res, flags = [], [], [], [], []
        self.slices = {}
        base = 0
        for o in objs:
            v = np.asarray(o.mesh.vertices, dtype=np.float64).reshape(-1, 3)
            f = np.asarray(o.mesh.faces, dtype=np.int64).reshape(-1, 3)
            tri_counts.append(len(f))
            tris.append(v[f].reshape(-1, 9))
            tr = o.transform
            xforms.append(np.concatenate([np.asarray(tr.translation, np.float64), np.asarray(tr.rotation, np.float64),
                                          np.asarray(tr.scale, np.float64)]))
            sm = sampled_meshes.get(o.object_id)
            take = o.object_id in inc and sm is not None and sm.total_samples > 0
            if sm is not None and len(sm.resolutions) == len(f):
                res.append(np.asarray(sm.resolutions, np.int64))
            else:
                res.append(np.ones(len(f), np.int64))
                take = False
            flags.append(1 if take else 0)
            if take:
                self.slices[o.object_id] = (base, base + int(sm.total_samples))
                base += int(sm.total_samples)
        self.n_samples = base
        self._keep = (np.ascontiguousarray(np.asarray(tri_counts, np.int64)),
                      np.ascontiguousarray(np.concatenate(tris) if tris else np.zeros((0, 9))),
                      np.ascontiguousarray(np.stack(xforms) if xforms else np.zeros((0, 10))),
                      np.ascontiguousarray(np.concatenate(res) if res else np.zeros(0, np.int64)),
                      np.ascontiguousarray(np.asarray(flags, np.uint8)))
        tc, tl, xf, rs, fl = self._keep
        _native.check(lib.gm_plan_set_scene(h, len(objs), _native.iptr(tc), _native.dptr(tl), _native.dptr(xf),
                                            _native.iptr(rs), _native.u8ptr(fl)), "gm_plan_set_scene")
        self._base_poses = xf.copy()
        self._obj_index = {o.object_id: i for i, o in enumerate(objs)}
        self._pose_key = ()
        n = int(lib.gm_plan_num_samples(h))
        if n != self.n_samples:
            raise RuntimeError(f"plan sample count {n} != layout total {self.n_samples}")
        self._keep = None
        self._owner = None  # _DeviceLink of the DensityMap whose values the accumulator holds

    def release(self) -> None:
        """Hand the device accumulator back: the linked map (accumulate_fixation)
        gets its values read back first if the device is ahead of it."""
        owner, self._owner = self._owner, None
        if owner is not None:
            owner.pull()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.gm_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    # ----------------------------------------------------------------- ops
    def accumulate(self, fixations, config: GenerationConfig, reset: bool = True, progress=None,
                   timers: Timings | None = None, batch: int = 0, flags: int = 0, _owner_ok: bool = False) -> None:
        """Add the fixations' contributions to the device values (`flags`:
        GmConfig.flags, e.g. _native.GM_FLAG_ONE_STREAM)."""
        if not _owner_ok:
            self.release()
        table = fixation_table(fixations)
        F = len(table)
        cfg = _native.GmConfig(float(config.theta), float(config.epsilon_abs), float(config.epsilon_rel),
                               int(config.zbuffer_resolution), int(bool(config.filtering_enabled)), int(batch),
                               int(flags))
        tm = _native.GmTimings()
        bad = np.zeros(1, np.int64)
        cb = _native.PROGRESS_FN(0)
        if progress is not None:
            state = {"n": 0}

            def _cb(done, total, _user):
                while state["n"] < done:
                    state["n"] += 1
                    progress(state["n"], total)

            cb = _native.PROGRESS_FN(_cb)
        rc = self._lib.gm_plan_accumulate(self._h, _native.dptr(table), F, ctypes.byref(cfg), int(bool(reset)),
                                          ctypes.byref(tm), cb, None, _native.iptr(bad))
        _native.check(rc, f"fixation {int(bad[0])}" if rc == _native.GM_ERR_INVALID_FRUSTUM else "gm_plan_accumulate")
        self.last_timings = tm
        if timers is not None:
            timers.add("cull", tm.cull_ms / 1e3)
            timers.add("rasterize", (tm.rasterize_ms + tm.texel_ms) / 1e3)
            timers.add("accumulate", (tm.mark_ms + tm.accumulate_ms) / 1e3)
            timers.add("setup", tm.setup_ms / 1e3)

    def set_overrides(self, overrides: dict | None) -> None:
        """Pose the scene for one fixation's overrides (object_id -> Transform;
        ids not in the scene are ignored, like _SampleCache.world and
        scene_world_triangles, reference density.py:121-127, raster.py:68-78);
        None/{} restores the base poses."""
        key = _pose_key(overrides, self._obj_index)
        if key == self._pose_key:
            return
        xf = self._base_poses.copy()
        for oid, t in (overrides or {}).items():
            i = self._obj_index.get(oid)
            if i is not None:
                xf[i] = _packed(t)
        _native.check(self._lib.gm_plan_set_poses(self._h, _native.dptr(np.ascontiguousarray(xf))),
                      "gm_plan_set_poses")
        self._pose_key = key

    def accumulate_log(self, fixations, config: GenerationConfig, reset: bool = True, progress=None,
                       timers: Timings | None = None, batch: int = 0, _owner_ok: bool = False) -> None:
        """accumulate() over a log that may carry pose overrides (dynamic
        scenes, reference density.py:123-127,161-165): the log is cut into
        runs of consecutive fixations with the same effective override set;
        each run is accumulated with the scene posed for it, in log order."""
        if not _owner_ok:
            self.release()
        table = fixation_table(fixations)
        ovs = _override_list(fixations)
        if ovs is None:
            self.set_overrides(None)
            self.accumulate(table, config, reset=reset, progress=progress, timers=timers, batch=batch,
                            _owner_ok=True)
            return
        F = len(table)
        keys = [_pose_key(o, self._obj_index) for o in ovs]
        try:
            a = 0
            first = True
            while a < F:
                b = a + 1
                while b < F and keys[b] == keys[a]:
                    b += 1
                self.set_overrides(ovs[a])
                cb = None
                if progress is not None:
                    cb = (lambda off: (lambda i, _t: progress(off + i, F)))(a)
                self.accumulate(table[a:b], config, reset=reset and first, progress=cb, timers=timers, batch=batch,
                                _owner_ok=True)
                first = False
                a = b
            if first and reset:
                self.accumulate(table[:0], config, reset=True, _owner_ok=True)
        finally:
            self.set_overrides(None)

    def global_max(self) -> float:
        out = np.zeros(1)
        _native.check(self._lib.gm_plan_max(self._h, _native.dptr(out)), "gm_plan_max")
        return float(out[0])

    def read(self, normalized_by: float | None = None) -> np.ndarray:
        out = np.empty(self.n_samples)
        if normalized_by is None:
            _native.check(self._lib.gm_plan_read(self._h, _native.dptr(out), None, 0.0), "gm_plan_read")
        else:
            _native.check(self._lib.gm_plan_read(self._h, None, _native.dptr(out), float(normalized_by)),
                          "gm_plan_read")
        return out

    def write(self, values: np.ndarray) -> None:
        self.release()
        v = np.ascontiguousarray(values, dtype=np.float64)
        _native.check(self._lib.gm_plan_write(self._h, _native.dptr(v)), "gm_plan_write")

    def values_device_ptr(self) -> int:
        return int(self._lib.gm_plan_values_device(self._h) or 0)

    def sync(self) -> None:
        _native.check(self._lib.gm_plan_sync(self._h), "gm_plan_sync")

    # multi-GPU: fused peer reduce of the ranks' partial maps (sharding.reduce_peers)
    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _native.check(self._lib.gm_plan_ipc_handle(self._h, buf), "gm_plan_ipc_handle")
        return buf.raw

    def open_peers(self, rank: int, world: int, handles: bytes) -> None:
        if len(handles) != 64 * world:
            raise ValueError("one 64-byte IPC handle per rank expected")
        _native.check(self._lib.gm_plan_open_peers(self._h, int(rank), int(world), handles), "gm_plan_open_peers")

    def reduce_peers(self) -> tuple:
        """Sum this rank's slice over the peers (rank order), store it into every
        peer's map; returns (slice max, device ms)."""
        mx = np.zeros(1)
        ms = ctypes.c_float(0.0)
        _native.check(self._lib.gm_plan_reduce_peers(self._h, _native.dptr(mx), ctypes.byref(ms)),
                      "gm_plan_reduce_peers")
        return float(mx[0]), float(ms.value)

    def split(self, flat: np.ndarray, sampled_meshes: dict) -> dict:
        """Per-object values: disjoint views of `flat` (a fresh buffer per call), no copy."""
        out = {}
        for oid, sm in sampled_meshes.items():
            if oid in self.slices:
                a, b = self.slices[oid]
                out[oid] = flat[a:b]
            else:
                out[oid] = np.zeros(sm.total_samples)
        return out

    def gather(self, values: dict) -> np.ndarray:
        flat = np.zeros(self.n_samples)
        for oid, (a, b) in self.slices.items():
            flat[a:b] = values[oid]
        return flat

    # ------------------------------------------------------- seam ports
    def depth_buffer(self, fixation, config: GenerationConfig, cull: bool = False) -> np.ndarray:
        """The (res, res) z-buffer kernels.rasterize produces for this fixation
        (crop frustum when filtering, else full), evaluated on the GPU."""
        row = fixation_table([fixation] if not isinstance(fixation, np.ndarray) else fixation[None, :])[0]
        res = int(config.zbuffer_resolution)
        out = np.empty((res, res))
        _native.check(self._lib.gm_plan_depth_buffer(self._h, _native.dptr(np.ascontiguousarray(row)),
                                                     float(config.theta), int(bool(config.filtering_enabled)), res,
                                                     int(not cull), _native.dptr(out)), "gm_plan_depth_buffer")
        return out

    def candidates(self, fixations, config: GenerationConfig, cap: int | None = None) -> list:
        """Per fixation, the sorted sample indices passing the NDC crop filter
        (kernels.py:302-319), computed by warp-ballot compaction on the GPU."""
        table = fixation_table(fixations)
        F = len(table)
        cap = self.n_samples if cap is None else cap
        out = np.zeros((max(F, 1), max(cap, 1)), np.int64)
        counts = np.zeros(max(F, 1), np.int64)
        _native.check(self._lib.gm_plan_candidates(self._h, _native.dptr(table), F, float(config.theta),
                                                   int(bool(config.filtering_enabled)),
                                                   int(config.zbuffer_resolution), _native.iptr(out), max(cap, 1),
                                                   _native.iptr(counts)), "gm_plan_candidates")
        return [np.sort(out[f, :min(int(counts[f]), cap)]) for f in range(F)]

    def positions(self) -> np.ndarray:
        out = np.empty((self.n_samples, 3))
        _native.check(self._lib.gm_plan_positions(self._h, _native.dptr(out)), "gm_plan_positions")
        return out


_PLANS: dict = {}
_PLAN_LIMIT = 4


def release_plans() -> None:
    """Destroy the cached ScenePlans (their device buffers are freed now, not at
    interpreter teardown, which CUDA may already have begun).  Runs at exit."""
    plans = list(_PLANS.values())
    _PLANS.clear()
    for plan in plans:
        plan.release()
        plan.__del__()


atexit.register(release_plans)


def get_plan(scene, sampled_meshes: dict, config: GenerationConfig, device: int = 0) -> ScenePlan:
    """Cached ScenePlan for (scene, layout, include list, device)."""
    included = _included_ids(scene, config)
    for oid in included:
        if oid not in sampled_meshes:
            raise KeyError(oid)
    key = (id(scene), id(sampled_meshes), tuple(included), device,
           tuple((oid, int(sm.total_samples)) for oid, sm in sampled_meshes.items()))
    plan = _PLANS.get(key)
    if plan is not None and plan.scene is scene and plan.sampled_meshes is sampled_meshes:
        return plan
    plan = ScenePlan(scene, sampled_meshes, included, device)
    if len(_PLANS) >= _PLAN_LIMIT:
        _PLANS.pop(next(iter(_PLANS)))
    _PLANS[key] = plan
    return plan


def _packed(t) -> np.ndarray:
    return np.concatenate([np.asarray(t.translation, np.float64).reshape(3), np.asarray(t.rotation, np.float64).reshape(4),
                           np.asarray(t.scale, np.float64).reshape(3)])


def _pose_key(overrides, index: dict) -> tuple:
    """Hashable identity of the poses an override dict imposes on the scene."""
    if not overrides:
        return ()
    return tuple(sorted((oid, _packed(t).tobytes()) for oid, t in overrides.items() if oid in index))


def _override_list(fixations):
    """Per-fixation override dicts, or None when the log has none at all."""
    if isinstance(fixations, np.ndarray):
        return None
    if getattr(fixations, "n_override_groups", None) == 0:  # FixationLog knows it parsed none
        return None
    ovs = [getattr(f, "overrides", None) or None for f in fixations]
    return ovs if any(o for o in ovs) else None


def generate(scene, sampled_meshes: dict, fixations, config: GenerationConfig, workers: int | None = None,
             progress=None, timers: Timings | None = None, device: int = 0, batch: int = 0) -> DensityMap:
    """All fixations, in log order, into a fresh un-normalized map.

    `fixations` is a list of Fixation objects (this package's or the
    reference's; pose overrides honoured) or an (F, 18) table in
    fixation-log column order.  `workers`
    is accepted for API compatibility; the GPU result does not depend on it.
    """
    config.validate()
    t0 = time.perf_counter()
    plan = get_plan(scene, sampled_meshes, config, device)
    t1 = time.perf_counter()
    plan.accumulate_log(fixations, config, reset=True, progress=progress, timers=timers, batch=batch)
    t2 = time.perf_counter()
    gmax = plan.global_max() if len(fixations) else 0.0
    t3 = time.perf_counter()
    values = plan.split(plan.read(), sampled_meshes)
    if timers is not None:  # wall-clock stages beside the device phases accumulate_log records
        timers.add("upload", t1 - t0)      # scene -> ScenePlan (first call for this scene only)
        timers.add("generate_wall", t2 - t1)
        timers.add("max", t3 - t2)
        timers.add("readback", time.perf_counter() - t3)
    return DensityMap(values, global_max=gmax, normalized=False)


class _DeviceLink:
    """Ties a DensityMap to the ScenePlan whose device accumulator holds its
    values, so a loop of accumulate_fixation calls runs as batched generation:

    * pending: fixations accepted by accumulate_fixation (validated on the host
      at the call, like the reference raises there) and not yet run; they run
      in log order, in batches, when PENDING_MAX are queued or when the map is
      observed -- reading `dmap.values` or `dmap.global_max`, or any other use
      of the plan.  The running max (reference density.py:180-194) is the max of
      the final values, since values only grow.
    * device_ahead: the plan holds newer values than the host arrays; reading
      `dmap.values` copies them back into those arrays (in place) first.
    * exposed: `dmap.values` was handed out since the last upload, so the
      caller may have edited the arrays: the next call re-uploads them.
    The plan remembers its owner link; before its accumulator is used for
    anything else (generate, another map) the owner is settled and read back."""

    PENDING_MAX = 8192

    def __init__(self, plan: "ScenePlan", dmap: DensityMap, config: GenerationConfig):
        self.plan = plan
        self.dmap_ref = weakref.ref(dmap)
        self.config = config
        self.key = _config_key(config)
        self.pending = []
        self.timers = None
        self.device_ahead = False
        self.exposed = False
        self.call_key = None  # (scene, layout, config, device) of the calls feeding it
        self.check = None     # _SetupCheck of that config
        self.rows = None      # the pending fixations' (F, 18) table rows, filled by the checks
        self.overrides = False  # a pending fixation carries pose overrides (then the objects are needed)

    def add(self, fixation) -> None:
        """Queue a fixation whose row the check has just built."""
        n = len(self.pending)
        if self.rows is None:
            self.rows = np.empty((self.PENDING_MAX, 18))
        self.rows[n] = self.check.row
        self.pending.append(fixation)
        if getattr(fixation, "overrides", None):
            self.overrides = True

    def flush(self) -> None:
        if not self.pending:
            return
        todo, self.pending = self.pending, []
        # no overrides: the table the per-call checks built (no per-object conversion)
        log = todo if self.overrides else self.rows[:len(todo)]
        self.overrides = False
        self.plan.accumulate_log(log, self.config, reset=False, timers=self.timers, _owner_ok=True)
        self.device_ahead = True
        dmap = self.dmap_ref()
        if dmap is not None and any(b > a for a, b in self.plan.slices.values()):
            d = object.__getattribute__(dmap, "__dict__")
            d["global_max"] = max(d["global_max"], self.plan.global_max())

    def pull(self, dmap: DensityMap | None = None) -> None:
        self.flush()
        dmap = dmap if dmap is not None else self.dmap_ref()
        if not self.device_ahead or dmap is None:
            self.device_ahead = False
            return
        self.device_ahead = False
        flat = self.plan.read()
        values = object.__getattribute__(dmap, "__dict__")["values"]
        for oid, (a, b) in self.plan.slices.items():
            values[oid][...] = flat[a:b]

    def expose(self, dmap: DensityMap) -> None:
        self.pull(dmap)
        self.exposed = True


def _config_key(config: GenerationConfig) -> tuple:
    return (float(config.theta), float(config.epsilon_abs), float(config.epsilon_rel), int(config.zbuffer_resolution),
            bool(config.filtering_enabled))


class _SetupCheck:
    """The host fixation setup of one fixation (gm_fixation_check) under the
    config's constants, computed once: accumulate_fixation's per-call check
    that the fixation's crop frustum is valid (the reference raises
    InvalidFrustumError from perspective_matrix at that call).  The row buffer
    and the raw function pointer are prebuilt; a call costs a few us."""

    def __init__(self, config: GenerationConfig):
        lib = _native.load()
        self.consts = ctypes.create_string_buffer(256)  # GmSetupConsts (< 256 bytes)
        res = int(config.zbuffer_resolution)
        lib.gm_setup_consts(float(config.theta), int(bool(config.filtering_enabled)), res, res, self.consts)
        self.row = np.zeros(18)
        self.views = (self.row[2:5], self.row[5:9], self.row[9:15], self.row[15:18])
        raw = ctypes.CDLL(str(lib._name)).gm_fixation_check  # no per-call argument conversion
        raw.restype = ctypes.c_int
        self.fn = raw
        self.args = (ctypes.c_void_p(self.row.ctypes.data), ctypes.cast(self.consts, ctypes.c_void_p))

    def __call__(self, f) -> None:
        r = self.row
        r[0] = f.start_time
        r[1] = f.duration
        pos, rot, fr, gz = self.views
        pos[...] = f.camera_position
        rot[...] = f.camera_rotation
        fr[...] = f.frustum
        gz[...] = f.gaze_dir
        rc = self.fn(*self.args)
        if rc:
            _native.check(rc, "fixation 0")


def accumulate_fixation(dmap: DensityMap, scene, sampled_meshes: dict, fixation, config: GenerationConfig,
                        cache=None, timers: Timings | None = None, device: int = 0) -> DensityMap:
    """Add one fixation to `dmap` in place (running max updated), return it
    (reference density.py:136-200).

    The map lives on the GPU while it is being fed (_DeviceLink): consecutive
    calls queue their fixations and run them as one batched generation when
    the map is next observed, so a loop over a log costs about one `generate`.
    A fixation whose crop frustum is degenerate raises InvalidFrustumError at
    its own call, as in the reference.  `timers` phases are recorded when the
    queued batch runs."""
    d = object.__getattribute__(dmap, "__dict__")
    link = d.get("_device_link")
    key = (id(scene), id(sampled_meshes), id(config), _config_key(config), device)
    if (link is not None and link.call_key == key and link.plan._owner is link and not link.exposed
            and (cache is None or cache is link.plan)):
        plan = link.plan  # the same map fed with the same scene / layout / config: no lookups
    else:
        config.validate()
        plan = cache if isinstance(cache, ScenePlan) else get_plan(scene, sampled_meshes, config, device)
        if (link is None or link.plan is not plan or plan._owner is not link or link.exposed
                or link.key != _config_key(config)):
            if link is not None:
                link.pull(dmap)
            plan.release()
            if d.get("_zero"):  # a fresh DensityMap.zeros: clear on the device, nothing to upload
                plan.accumulate(np.zeros((0, 18)), config, reset=True, _owner_ok=True)
            else:
                plan.write(plan.gather(d["values"]))
            link = _DeviceLink(plan, dmap, config)
            d["_device_link"] = link
            plan._owner = link
        link.config = config
        link.call_key = key
        link.check = _SetupCheck(config)
    link.check(fixation)  # raises InvalidFrustumError here, as the reference does
    if timers is not None:
        link.timers = timers
    link.add(fixation)
    if len(link.pending) >= link.PENDING_MAX:
        link.flush()
    return dmap


def normalize(dmap: DensityMap, timers: Timings | None = None, device: int = 0) -> DensityMap:
    """values / global_max on the GPU into a new map; idempotent, zero-safe."""
    t0 = time.perf_counter()
    if dmap.normalized or dmap.global_max <= 0.0:
        out = dmap.copy()
        out.normalized = True
    else:
        keys = list(dmap.values)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(dmap.values[k], np.float64) for k in keys])
                                    if keys else np.zeros(0))
        res = np.empty_like(flat)
        if len(flat):
            lib = _native.load()
            _native.check(lib.gm_normalize(device, _native.dptr(flat), len(flat), float(dmap.global_max),
                                           _native.dptr(res)), "gm_normalize")
        vals, o = {}, 0
        for k in keys:
            n = len(dmap.values[k])
            vals[k] = res[o:o + n]
            o += n
        out = DensityMap(vals, global_max=1.0, normalized=True)
    if timers is not None:
        timers.add("normalize", time.perf_counter() - t0)
    return out
