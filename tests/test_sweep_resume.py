"""The sweep harness's JSONL checkpoint (scripts/design_rules.py): a sweep
interrupted part-way and restarted measures only the schedules it had not
recorded, reuses the recorded times in order, and ignores a torn last line
or a line whose schedule text no longer matches its index."""
import importlib.util
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _harness():
    pytest.importorskip("torch")
    spec = importlib.util.spec_from_file_location("design_rules", os.path.join(ROOT, "scripts", "design_rules.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_resume_skips_measured_schedules(tmp_path):
    m = _harness()
    from paper_2203_02530_b200 import schedules as PS
    space = PS.enumerate_derived(2)[:40]
    calls = []

    def measure(ops):
        calls.append(PS.describe(ops))
        return 1e-6 * (len(calls) + 0.5)

    path = str(tmp_path / "sweep.jsonl")

    class Stop(Exception):
        pass

    def measure_until(ops):
        if len(calls) == 25:
            raise Stop()
        return measure(ops)
    with pytest.raises(Stop):
        m.sweep_with_resume(space, measure_until, path)
    lines = open(path).read().splitlines()
    assert len(lines) == 25
    # a torn last line and a stale line (wrong schedule text for its index)
    with open(path, "a") as f:
        f.write('{"i": 25, "sch')
    rec = [json.loads(l) for l in lines]
    rec[3]["schedule"] = "stale"
    with open(path, "w") as f:
        f.write("\n".join(json.dumps(r) for r in rec) + "\n" + '{"i": 25, "sch')
    first = [r["t"] for r in rec]
    times, reused = m.sweep_with_resume(space, measure, path)
    assert reused == 24 and len(times) == 40
    assert len(calls) == 25 + 16                       # schedule 3 and the 15 unmeasured ones
    assert np.allclose(times[:3], first[:3]) and np.allclose(times[4:25], first[4:25])
    # every line written after the torn one parses: a third run measures nothing
    calls.clear()
    times2, reused2 = m.sweep_with_resume(space, measure, path)
    assert reused2 == 40 and not calls and np.allclose(times2, times)
