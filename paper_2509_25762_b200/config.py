"""JSON run configuration with the reference's schema.

Mirrors ``rlpipe::load_config_text`` / ``config_echo`` /
``RunConfig::task_fingerprint`` / ``RunConfig::baseline``
(``proj/core/src/config.cpp:75-250``, ``:253-290``, ``:306-409``, ``:411-420``):

* the same keys, presets (``desk`` | ``paper``, config.cpp:88-98), enums and
  defaults (``config.hpp:28-77``, ``model.hpp:43-81``, ``ppo.hpp:11-17``,
  ``delayed_sgd.hpp:17-31``);
* the same value coercions as ``nlohmann::json::get<T>`` (numbers convert
  to numeric fields, booleans only to ``int`` ones, ``bool`` / ``string`` /
  arrays must have that JSON type; out-of-range float -> int casts as gcc
  emits them on x86-64);
* the same error behaviour: every schema problem is collected and reported as
  one ``ConfigError("config rejected:\\n  - ...")`` (config.cpp:233-237);
  only a config that passes the schema is validated (config.cpp:253-290,
  nested ``validate()`` messages of model.cpp:10-47, ppo.cpp:10-16,
  delayed_sgd.cpp:9-27);
* ``config_echo`` in the layout of stock ``ordered_json::dump(2)`` (the
  cudnn_frontend copy of nlohmann this image builds the reference with prints
  integer arrays inline; the tests compare echoes structurally) and
  ``task_fingerprint`` = FNV-1a of the compact dump without the scheduler
  knobs, so fingerprints computed here and by the reference agree.

Extension (ours, not in the reference schema): optional ``model`` and ``gpu``
blocks naming the engine shapes and the SM split (``load_config_text(...,
extended=True)``); they are not part of the echo or the fingerprint.

Invalid JSON raises ``ConfigError("config is not valid JSON: ...")`` like the
reference; the parser's own message after the prefix differs.
"""
import copy
import json
import math

from . import abi
from . import scheduler as S


class ConfigError(ValueError):
    """rlpipe::ConfigError (errors.hpp:9-13)."""


def defaults():
    """RunConfig{} (config.hpp:28-77) as a plain dict."""
    return dict(
        mode=0, steps=100, seeds=[1], out_dir="out", batch_size=8, prompt_len=8, prompt_count=-1,
        delta_init=0, delta_min=0, delta_max=8, controller=0, window=8, delta_inc=1, delta_dec=1,
        chunk_size=256, schedule_mode=0, tune_chunks=False, chunk_candidates=[128, 256, 512],
        retune_period=50,
        latency=dict(decode_per_token=1, prefill_per_token=1, reward_residual=0, chunk_switch_cost=0,
                     transfer_per_chunk=0, placement=1, count_prompt_in_prefill=True),
        lengths=dict(kind=0, fast_len=100, slow_len=600, p_slow=0.0, mu_log=5.0, sigma_log=0.8,
                     cap=4096, table=[]),
        ppo=dict(gamma=1.0, **{"lambda": 1.0}, clip_epsilon=0.2, learning_rate=0.1,
                 value_learning_rate=0.2),
        vocab=4, target_token=0, reward_scale=1.0, reward_bias=0.0,
        sgd=dict(dim=10, mu=0.1, lipschitz=1.0, eta=1.0 / 1.1, d_max=0.0, g_max=64.0, iterations=10000,
                 initial_distance_sq=25.0, noise=1, eigenvalues=[]),
        reward_proxy=dict(kind=0, value=1.0, ramp_scale=1.0, ramp_steps=100),
        fail_after_step=-1,
        model=None, gpu=None)


# ------------------------------------------------------ nlohmann get<T> rules
class _Wrong(Exception):
    pass


def _wrap(v, bits, signed):
    v &= (1 << bits) - 1
    if signed and v >= 1 << (bits - 1):
        v -= 1 << bits
    return v


def _num(v, allow_bool):
    """nlohmann's from_json for int64_t / uint64_t / double (its own
    number_*_t types: get_arithmetic_value) takes numbers only; the generic
    arithmetic overload (int here) also takes booleans."""
    if isinstance(v, bool):
        if allow_bool:
            return int(v)
        raise _Wrong()
    if isinstance(v, (int, float)):
        return v
    raise _Wrong()


def _float_to_int(x, bits, signed):
    """static_cast<int{32,64}_t / uint64_t>(double) as gcc emits it for
    x86-64 (cvttsd2si; out-of-range values give the "integer indefinite"
    0x80..0; uint64 goes through the 2^63 split)."""
    t = math.trunc(x)
    if signed:
        lo = -(1 << (bits - 1))
        return t if lo <= t < -lo else lo
    if t >= 1 << 64:
        return 0
    if t >= 1 << 63:
        return t
    if t >= -(1 << 63):
        return t & ((1 << 64) - 1)
    return 1 << 63


def _int(bits=32, signed=True):
    def conv(v):
        x = _num(v, bits == 32)
        if isinstance(x, float):
            return _float_to_int(x, bits, signed)
        return _wrap(x, bits, signed)
    return conv


def _double(v):
    return float(_num(v, False))


def _bool(v):
    if not isinstance(v, bool):
        raise _Wrong()
    return v


def _string(v):
    if not isinstance(v, str):
        raise _Wrong()
    return v


def _vector(elem):
    def conv(v):
        if not isinstance(v, list):
            raise _Wrong()
        return [elem(x) for x in v]
    return conv


def _pair_int_double(v):
    if not isinstance(v, list) or len(v) < 2:
        raise _Wrong()
    return (_int()(v[0]), _double(v[1]))


I32, I64, U64 = _int(), _int(64), _int(64, False)


class _Schema:
    """config.cpp:17-73."""

    def __init__(self):
        self.errors = []

    def fail(self, msg):
        self.errors.append(msg)

    def check_keys(self, obj, scope, allowed):
        for key in obj:
            if key not in allowed:
                self.fail(f"unknown key '{scope}{key}'")

    def read(self, obj, scope, key, conv, dst, field):
        if key not in obj:
            return
        try:
            dst[field] = conv(obj[key])
        except _Wrong:
            self.fail(f"key '{scope}{key}' has the wrong type")

    def read_enum(self, obj, scope, key, values, dst, field):
        if key not in obj:
            return
        v = obj[key]
        if not isinstance(v, str):
            self.fail(f"key '{scope}{key}' must be a string")
            return
        for name, code in values:
            if v == name:
                dst[field] = code
                return
        self.fail(f"key '{scope}{key}' must be one of " + "|".join(n for n, _ in values))


class _Items(dict):
    """A non-object block seen through nlohmann's items(): an array yields the
    keys "0".."n-1", a scalar one key "", null none; contains() is false for
    all of them, so no field is read."""

    def __init__(self, keys):
        super().__init__()
        self.keys_ = keys

    def __iter__(self):
        return iter(self.keys_)

    def __contains__(self, key):
        return False


def _obj(root, key, s, scope):
    """root.at(key) as the reference uses it (check_keys over items(), reads
    through contains())."""
    v = root[key]
    if isinstance(v, dict):
        return v
    if isinstance(v, list):
        return _Items([str(i) for i in range(len(v))])
    return _Items([] if v is None else [""])


MODES = [("simulate", 0), ("train", 1), ("tune", 2)]
CONTROLLERS = [("fixed", 0), ("alg1", 1), ("eq4", 2)]
SCHEDULES = [("streamed", 0), ("sequential", 1)]
PLACEMENTS = [("colocated", 0), ("disaggregated", 1)]
LENGTH_KINDS = [("two_point", 0), ("lognormal", 1), ("empirical", 2)]
NOISES = [("none", 0), ("random_unit", 1), ("outward", 2)]
PROXY_KINDS = [("constant", 0), ("ramp", 1)]


def _parse(root, extended):
    """parse (config.cpp:75-239)."""
    s = _Schema()
    c = defaults()
    top = ["schema_version", "preset", "mode", "steps", "seeds", "out_dir", "batch", "delta", "chunk",
           "latency", "lengths", "ppo", "sgd", "reward_proxy", "debug"]
    s.check_keys(root, "", top + (["model", "gpu"] if extended else []))
    tmp = {}
    s.read(root, "", "schema_version", I32, tmp, "v")
    if tmp.get("v", 1) != 1:
        s.fail("schema_version must be 1")
    s.read(root, "", "preset", _string, tmp, "preset")
    preset = tmp.get("preset", "desk")
    if preset == "paper":
        c.update(batch_size=112, chunk_size=256, chunk_candidates=[128, 256, 512], retune_period=50)
    elif preset != "desk":
        s.fail("preset must be desk|paper")
    s.read_enum(root, "", "mode", MODES, c, "mode")
    s.read(root, "", "steps", I32, c, "steps")
    s.read(root, "", "seeds", _vector(U64), c, "seeds")
    s.read(root, "", "out_dir", _string, c, "out_dir")
    if "batch" in root:
        b = _obj(root, "batch", s, "batch.")
        s.check_keys(b, "batch.", ["size", "prompt_len", "prompts"])
        s.read(b, "batch.", "size", I32, c, "batch_size")
        s.read(b, "batch.", "prompt_len", I32, c, "prompt_len")
        s.read(b, "batch.", "prompts", I64, c, "prompt_count")
    if "delta" in root:
        d = _obj(root, "delta", s, "delta.")
        s.check_keys(d, "delta.", ["init", "min", "max", "controller", "window", "inc", "dec"])
        s.read(d, "delta.", "init", I32, c, "delta_init")
        s.read(d, "delta.", "min", I32, c, "delta_min")
        s.read(d, "delta.", "max", I32, c, "delta_max")
        s.read_enum(d, "delta.", "controller", CONTROLLERS, c, "controller")
        s.read(d, "delta.", "window", I32, c, "window")
        s.read(d, "delta.", "inc", I32, c, "delta_inc")
        s.read(d, "delta.", "dec", I32, c, "delta_dec")
    if "chunk" in root:
        k = _obj(root, "chunk", s, "chunk.")
        s.check_keys(k, "chunk.", ["size", "mode", "tune", "candidates", "retune_period"])
        s.read(k, "chunk.", "size", I32, c, "chunk_size")
        s.read_enum(k, "chunk.", "mode", SCHEDULES, c, "schedule_mode")
        s.read(k, "chunk.", "tune", _bool, c, "tune_chunks")
        s.read(k, "chunk.", "candidates", _vector(I32), c, "chunk_candidates")
        s.read(k, "chunk.", "retune_period", I32, c, "retune_period")
    if "latency" in root:
        lt, L = _obj(root, "latency", s, "latency."), c["latency"]
        s.check_keys(lt, "latency.", ["decode_per_token", "prefill_per_token", "reward_residual",
                                      "chunk_switch_cost", "transfer_per_chunk", "placement",
                                      "count_prompt_in_prefill"])
        for key in ("decode_per_token", "prefill_per_token", "reward_residual", "chunk_switch_cost",
                    "transfer_per_chunk"):
            s.read(lt, "latency.", key, I64, L, key)
        s.read_enum(lt, "latency.", "placement", PLACEMENTS, L, "placement")
        s.read(lt, "latency.", "count_prompt_in_prefill", _bool, L, "count_prompt_in_prefill")
    if "lengths" in root:
        ln, D = _obj(root, "lengths", s, "lengths."), c["lengths"]
        s.check_keys(ln, "lengths.", ["kind", "fast_len", "slow_len", "p_slow", "mu_log", "sigma_log",
                                      "cap", "table"])
        s.read_enum(ln, "lengths.", "kind", LENGTH_KINDS, D, "kind")
        s.read(ln, "lengths.", "fast_len", I32, D, "fast_len")
        s.read(ln, "lengths.", "slow_len", I32, D, "slow_len")
        s.read(ln, "lengths.", "p_slow", _double, D, "p_slow")
        s.read(ln, "lengths.", "mu_log", _double, D, "mu_log")
        s.read(ln, "lengths.", "sigma_log", _double, D, "sigma_log")
        s.read(ln, "lengths.", "cap", I32, D, "cap")
        s.read(ln, "lengths.", "table", _vector(_pair_int_double), D, "table")
    if "ppo" in root:
        p, P = _obj(root, "ppo", s, "ppo."), c["ppo"]
        s.check_keys(p, "ppo.", ["gamma", "lambda", "clip_epsilon", "learning_rate", "value_learning_rate",
                                 "vocab", "target_token", "reward_scale", "reward_bias"])
        for key in ("gamma", "lambda", "clip_epsilon", "learning_rate", "value_learning_rate"):
            s.read(p, "ppo.", key, _double, P, key)
        s.read(p, "ppo.", "vocab", I32, c, "vocab")
        s.read(p, "ppo.", "target_token", I32, c, "target_token")
        s.read(p, "ppo.", "reward_scale", _double, c, "reward_scale")
        s.read(p, "ppo.", "reward_bias", _double, c, "reward_bias")
    if "sgd" in root:
        g, G = _obj(root, "sgd", s, "sgd."), c["sgd"]
        s.check_keys(g, "sgd.", ["dim", "mu", "lipschitz", "eta", "d_max", "g_max", "iterations",
                                 "initial_distance_sq", "noise", "eigenvalues"])
        s.read(g, "sgd.", "dim", I32, G, "dim")
        for key in ("mu", "lipschitz", "eta", "d_max", "g_max"):
            s.read(g, "sgd.", key, _double, G, key)
        s.read(g, "sgd.", "iterations", I64, G, "iterations")
        s.read(g, "sgd.", "initial_distance_sq", _double, G, "initial_distance_sq")
        s.read_enum(g, "sgd.", "noise", NOISES, G, "noise")
        s.read(g, "sgd.", "eigenvalues", _vector(_double), G, "eigenvalues")
    if "reward_proxy" in root:
        r, R = _obj(root, "reward_proxy", s, "reward_proxy."), c["reward_proxy"]
        s.check_keys(r, "reward_proxy.", ["kind", "value", "ramp_scale", "ramp_steps"])
        s.read_enum(r, "reward_proxy.", "kind", PROXY_KINDS, R, "kind")
        s.read(r, "reward_proxy.", "value", _double, R, "value")
        s.read(r, "reward_proxy.", "ramp_scale", _double, R, "ramp_scale")
        s.read(r, "reward_proxy.", "ramp_steps", I32, R, "ramp_steps")
    if "debug" in root:
        d = _obj(root, "debug", s, "debug.")
        s.check_keys(d, "debug.", ["fail_after_step"])
        s.read(d, "debug.", "fail_after_step", I32, c, "fail_after_step")
    if extended:
        _parse_extension(root, s, c)
    if s.errors:
        raise ConfigError("config rejected:" + "".join("\n  - " + e for e in s.errors))
    validate(c)
    return c


def _parse_extension(root, s, c):
    """Our `model` / `gpu` blocks: engine shapes (names of engine.SHAPES or
    explicit dims) and the GPU step settings."""
    if "model" in root:
        m = _obj(root, "model", s, "model.")
        s.check_keys(m, "model.", ["actor", "reward", "critic", "ref"])
        c["model"] = {}
        for role in ("actor", "reward", "critic", "ref"):
            if role in m:
                v = m[role]
                if isinstance(v, str) or (isinstance(v, dict) and all(isinstance(x, int) for x in v.values())):
                    c["model"][role] = v
                else:
                    s.fail(f"key 'model.{role}' must be a shape name or an object of integer dims")
    if "gpu" in root:
        g = _obj(root, "gpu", s, "gpu.")
        s.check_keys(g, "gpu.", ["dtype", "scorer_sms", "carry", "kl_coef", "whiten"])
        c["gpu"] = dict(dtype=abi.DTYPE_BF16, scorer_sms=0, carry=abi.CARRY_TOKEN, kl_coef=0.05, whiten=True)
        s.read_enum(g, "gpu.", "dtype", [("f32", abi.DTYPE_F32), ("bf16", abi.DTYPE_BF16)], c["gpu"], "dtype")
        s.read(g, "gpu.", "scorer_sms", I32, c["gpu"], "scorer_sms")
        s.read_enum(g, "gpu.", "carry", [("chunk", abi.CARRY_CHUNK), ("token", abi.CARRY_TOKEN)], c["gpu"],
                    "carry")
        s.read(g, "gpu.", "kl_coef", _double, c["gpu"], "kl_coef")
        s.read(g, "gpu.", "whiten", _bool, c["gpu"], "whiten")


def _validate_nested(c):
    L, D, P, G = c["latency"], c["lengths"], c["ppo"], c["sgd"]

    def latency():  # model.cpp:10-15
        if min(L["decode_per_token"], L["prefill_per_token"], L["reward_residual"], L["chunk_switch_cost"],
               L["transfer_per_chunk"]) < 0:
            raise ConfigError("latency model: all tick costs must be >= 0")

    def lengths():  # model.cpp:17-47
        if D["cap"] < 1:
            raise ConfigError("length distribution: cap must be >= 1")
        if D["kind"] == 0:
            if D["fast_len"] < 1 or D["slow_len"] < 1:
                raise ConfigError("two-point lengths must be >= 1")
            if D["fast_len"] > D["cap"] or D["slow_len"] > D["cap"]:
                raise ConfigError("two-point lengths must be <= cap")
            if D["p_slow"] < 0.0 or D["p_slow"] > 1.0:
                raise ConfigError("two-point p_slow must be in [0,1]")
        elif D["kind"] == 1:
            if D["sigma_log"] < 0.0:
                raise ConfigError("lognormal sigma must be >= 0")
        else:
            if not D["table"]:
                raise ConfigError("empirical table must be non-empty")
            total = 0.0
            for ln, w in D["table"]:
                if ln < 1 or ln > D["cap"]:
                    raise ConfigError("empirical table lengths must be in [1, cap]")
                if w < 0.0:
                    raise ConfigError("empirical table weights must be >= 0")
                total += w
            if total <= 0.0:
                raise ConfigError("empirical table needs positive total weight")

    def ppo():  # ppo.cpp:10-16
        if P["gamma"] < 0.0 or P["gamma"] > 1.0:
            raise ConfigError("gamma must be in [0,1]")
        if P["lambda"] < 0.0 or P["lambda"] > 1.0:
            raise ConfigError("lambda must be in [0,1]")
        if not P["clip_epsilon"] > 0.0:
            raise ConfigError("clip epsilon must be > 0")
        if not P["learning_rate"] > 0.0:
            raise ConfigError("learning rate must be > 0")
        if not P["value_learning_rate"] > 0.0:
            raise ConfigError("value learning rate must be > 0")

    def sgd():  # delayed_sgd.cpp:9-27
        if G["dim"] < 1:
            raise ConfigError("delayed-sgd dimension must be >= 1")
        if not G["mu"] > 0.0 or not G["mu"] <= G["lipschitz"]:
            raise ConfigError("delayed-sgd requires 0 < mu <= L")
        if not G["eta"] > 0.0 or G["eta"] > 1.0 / (G["lipschitz"] + G["mu"]):
            raise ConfigError("delayed-sgd requires 0 < eta <= 1/(L+mu)")
        if G["d_max"] < 0.0 or G["g_max"] < 0.0:
            raise ConfigError("delayed-sgd norm bounds must be >= 0")
        if G["iterations"] < 0:
            raise ConfigError("delayed-sgd iterations must be >= 0")
        if not G["initial_distance_sq"] > 0.0:
            raise ConfigError("delayed-sgd initial distance must be > 0")
        if G["eigenvalues"]:
            if len(G["eigenvalues"]) != G["dim"]:
                raise ConfigError("delayed-sgd spectrum size must match dim")
            for ev in G["eigenvalues"]:
                if ev < G["mu"] or ev > G["lipschitz"]:
                    raise ConfigError("delayed-sgd spectrum must lie within [mu, L]")

    return [latency, lengths, ppo, sgd]


def validate(c):
    """RunConfig::validate (config.cpp:253-290)."""
    e = []
    if c["steps"] < 1:
        e.append("steps must be >= 1")
    if not c["seeds"]:
        e.append("seeds must be non-empty")
    if c["batch_size"] < 1:
        e.append("batch.size must be >= 1")
    if c["prompt_len"] < 1:
        e.append("batch.prompt_len must be >= 1")
    if c["delta_min"] > c["delta_max"]:
        e.append(f"delta.min ({c['delta_min']}) must be <= delta.max ({c['delta_max']})")
    if c["delta_min"] < 0:
        e.append("delta.min must be >= 0")
    if c["delta_init"] < c["delta_min"] or c["delta_init"] > c["delta_max"]:
        e.append("delta.init must lie within [delta.min, delta.max]")
    if c["window"] < 1:
        e.append("delta.window must be >= 1")
    if c["delta_inc"] < 1 or c["delta_dec"] < 1:
        e.append("delta momenta must be >= 1")
    if c["chunk_size"] < 1:
        e.append("chunk.size must be >= 1")
    if c["retune_period"] < 1:
        e.append("chunk.retune_period must be >= 1")
    if c["tune_chunks"]:
        if not c["chunk_candidates"]:
            e.append("chunk.candidates must be non-empty when tuning")
        for x in c["chunk_candidates"]:
            if x < 1:
                e.append("chunk.candidates must all be >= 1")
        if c["retune_period"] < len(c["chunk_candidates"]):
            e.append("chunk.retune_period must cover one step per candidate")
    if c["vocab"] < 2 or c["vocab"] > 16:
        e.append("ppo.vocab must be in [2,16]")
    if c["target_token"] < 0 or c["target_token"] >= c["vocab"]:
        e.append("ppo.target_token must be a vocabulary token")
    for check in _validate_nested(c):
        try:
            check()
        except ConfigError as x:
            e.append(str(x))
    if e:
        raise ConfigError("config rejected:" + "".join("\n  - " + m for m in e))


def _no_constants(name):
    raise ValueError(f"invalid literal {name}")


def load_config_text(text, extended=False):
    """load_config_text (config.cpp:302-312)."""
    try:
        root = json.loads(text, parse_constant=_no_constants)
    except ValueError as e:
        raise ConfigError(f"config is not valid JSON: {e}") from None
    if not isinstance(root, dict):
        raise ConfigError("config root must be a JSON object")
    return _parse(root, extended)


def load_config(path, extended=False):
    """load_config (config.cpp:294-300)."""
    try:
        with open(path, encoding="utf-8") as f:
            text = f.read()
    except OSError:
        raise ConfigError(f"cannot open config file: {path}") from None
    return load_config_text(text, extended)


def baseline(c):
    """RunConfig::baseline (config.cpp:411-420)."""
    b = copy.deepcopy(c)
    b.update(delta_init=0, delta_min=0, delta_max=0, controller=0, schedule_mode=1, tune_chunks=False)
    return b


def _name(table, code):
    return next(n for n, v in table if v == code)


def echo_obj(c):
    """echo_json (config.cpp:316-388), key order included."""
    L, D, P, G, R = c["latency"], c["lengths"], c["ppo"], c["sgd"], c["reward_proxy"]
    return {
        "schema_version": 1, "mode": _name(MODES, c["mode"]), "steps": c["steps"], "seeds": list(c["seeds"]),
        "out_dir": c["out_dir"],
        "batch": {"size": c["batch_size"], "prompt_len": c["prompt_len"], "prompts": c["prompt_count"]},
        "delta": {"init": c["delta_init"], "min": c["delta_min"], "max": c["delta_max"],
                  "controller": _name(CONTROLLERS, c["controller"]), "window": c["window"],
                  "inc": c["delta_inc"], "dec": c["delta_dec"]},
        "chunk": {"size": c["chunk_size"], "mode": _name(SCHEDULES, c["schedule_mode"]),
                  "tune": bool(c["tune_chunks"]), "candidates": list(c["chunk_candidates"]),
                  "retune_period": c["retune_period"]},
        "latency": {"decode_per_token": L["decode_per_token"], "prefill_per_token": L["prefill_per_token"],
                    "reward_residual": L["reward_residual"], "chunk_switch_cost": L["chunk_switch_cost"],
                    "transfer_per_chunk": L["transfer_per_chunk"],
                    "placement": _name(PLACEMENTS, L["placement"]),
                    "count_prompt_in_prefill": bool(L["count_prompt_in_prefill"])},
        "lengths": {"kind": _name(LENGTH_KINDS, D["kind"]), "fast_len": D["fast_len"], "slow_len": D["slow_len"],
                    "p_slow": float(D["p_slow"]), "mu_log": float(D["mu_log"]),
                    "sigma_log": float(D["sigma_log"]), "cap": D["cap"],
                    "table": [[ln, float(w)] for ln, w in D["table"]]},
        "ppo": {"gamma": float(P["gamma"]), "lambda": float(P["lambda"]), "clip_epsilon": float(P["clip_epsilon"]),
                "learning_rate": float(P["learning_rate"]),
                "value_learning_rate": float(P["value_learning_rate"]), "vocab": c["vocab"],
                "target_token": c["target_token"], "reward_scale": float(c["reward_scale"]),
                "reward_bias": float(c["reward_bias"])},
        "sgd": {"dim": G["dim"], "mu": float(G["mu"]), "lipschitz": float(G["lipschitz"]), "eta": float(G["eta"]),
                "d_max": float(G["d_max"]), "g_max": float(G["g_max"]), "iterations": G["iterations"],
                "initial_distance_sq": float(G["initial_distance_sq"]), "noise": _name(NOISES, G["noise"]),
                "eigenvalues": [float(x) for x in G["eigenvalues"]]},
        "reward_proxy": {"kind": _name(PROXY_KINDS, R["kind"]), "value": float(R["value"]),
                         "ramp_scale": float(R["ramp_scale"]), "ramp_steps": R["ramp_steps"]},
    }


def config_echo(c):
    """config_echo (config.cpp:392): ordered_json::dump(2) + newline."""
    return json.dumps(echo_obj(c), indent=2, ensure_ascii=False) + "\n"


def task_fingerprint(c):
    """RunConfig::task_fingerprint (config.cpp:394-409): FNV-1a (64-bit) of the
    compact dump without delta / chunk / seeds / out_dir, as 16 hex digits."""
    j = echo_obj(c)
    for k in ("delta", "chunk", "seeds", "out_dir"):
        del j[k]
    h = 0xcbf29ce484222325
    for b in json.dumps(j, separators=(",", ":"), ensure_ascii=False).encode("utf-8"):
        h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def to_run_config(c):
    """The C ABI's oppo_run_config (run_seed's input) for a parsed config."""
    L, D, P, R = c["latency"], c["lengths"], c["ppo"], c["reward_proxy"]
    if len(c["chunk_candidates"]) > abi.MAX_CANDIDATES or len(D["table"]) > abi.MAX_TABLE:
        raise ConfigError("config exceeds the C ABI's candidate / length-table capacity")
    cfg = S.default_config(
        mode=c["mode"], steps=c["steps"], batch_size=c["batch_size"], prompt_len=c["prompt_len"],
        prompt_count=c["prompt_count"], delta_init=c["delta_init"], delta_min=c["delta_min"],
        delta_max=c["delta_max"], controller=c["controller"], window=c["window"], delta_inc=c["delta_inc"],
        delta_dec=c["delta_dec"], chunk_size=c["chunk_size"], schedule_mode=c["schedule_mode"],
        tune_chunks=int(c["tune_chunks"]), chunk_candidates=c["chunk_candidates"],
        retune_period=c["retune_period"], vocab=c["vocab"], target_token=c["target_token"],
        reward_scale=c["reward_scale"], reward_bias=c["reward_bias"], proxy_kind=R["kind"],
        proxy_ramp_steps=R["ramp_steps"], proxy_value=R["value"], proxy_ramp_scale=R["ramp_scale"],
        fail_after_step=c["fail_after_step"],
        latency_decode_per_token=L["decode_per_token"], latency_prefill_per_token=L["prefill_per_token"],
        latency_reward_residual=L["reward_residual"], latency_chunk_switch_cost=L["chunk_switch_cost"],
        latency_transfer_per_chunk=L["transfer_per_chunk"], latency_placement=L["placement"],
        latency_count_prompt_in_prefill=int(L["count_prompt_in_prefill"]),
        lengths_kind=D["kind"], lengths_fast_len=D["fast_len"], lengths_slow_len=D["slow_len"],
        lengths_p_slow=D["p_slow"], lengths_mu_log=D["mu_log"], lengths_sigma_log=D["sigma_log"],
        lengths_cap=D["cap"], lengths_table=D["table"],
        ppo_gamma=P["gamma"], ppo_lambda=P["lambda"], ppo_clip_epsilon=P["clip_epsilon"],
        ppo_learning_rate=P["learning_rate"], ppo_value_learning_rate=P["value_learning_rate"])
    return cfg


__all__ = ["ConfigError", "defaults", "load_config", "load_config_text", "validate", "baseline",
           "config_echo", "task_fingerprint", "to_run_config", "echo_obj"]
