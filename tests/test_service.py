"""The SSE session service (paper_2511_20426_b200/service.py)
with the reference gateway's behaviour (reference pkg/tests/test_gateway.py):
live stream == trace replay, block payloads, seq order, late / mid-run
subscribers, and the HTTP routes with their status codes.  CPU tests drive
it through the engine seam with the CPU oracle forward; the -m gpu test runs
the device engine."""

import base64
import json
import threading
import time

import numpy as np
import pytest

from paper_2511_20426_b200 import CascadeConfig, with_fields
from paper_2511_20426_b200.service import SessionManager, create_app
from paper_2511_20426_b200.stream import events_from_trace


@pytest.fixture(scope="module")
def service_config():
    return CascadeConfig(total_frames=39, workers=2, pass_cost_base=1.0)


def _finished(manager, config, prompt="a red cube"):
    s = manager.create(config, prompt, start=False)
    s.thread.start()
    s.thread.join()
    assert s.status == "done", s.error
    return s


def test_live_stream_equals_trace_replay(oracle_engine, service_config):
    m = SessionManager()
    s = m.create(service_config, "a red cube", start=False)
    got = []
    t = threading.Thread(target=lambda: got.extend(s.log.subscribe()))
    t.start()
    s.thread.start()
    s.thread.join()
    t.join()
    assert got == events_from_trace(s.result.trace, service_config, s.result.outputs)


def test_block_payload_and_seq(oracle_engine, service_config):
    s = _finished(SessionManager(), service_config)
    docs = [json.loads(l) for l in events_from_trace(s.result.trace, service_config, s.result.outputs)]
    blocks = [d for d in docs if d["type"] == "block"]
    assert [b["index"] for b in blocks] == list(range(13))
    px = np.frombuffer(base64.b64decode(blocks[0]["pixels"]["data"]), dtype="<f4")
    assert px.reshape(blocks[0]["pixels"]["shape"]).shape == (12, 16)
    assert blocks[0]["video_frames"] == 12 and blocks[0]["fps"] > 0
    assert [d["seq"] for d in docs] == list(range(len(docs)))
    assert docs[-1]["type"] == "done" and docs[-1]["blocks"] == 13
    first = next(i for i, d in enumerate(docs) if d["type"] == "block")
    assert sum(d["type"] == "metrics" for d in docs[:first]) == service_config.passes - 1
    assert s.snapshot()["blocks_emitted"] == 13


def test_two_subscribers_identical(oracle_engine, service_config):
    m = SessionManager()
    s = m.create(with_fields(service_config, total_frames=15), "p", start=False)
    a, b = [], []
    ts = [threading.Thread(target=lambda out=out: out.extend(s.log.subscribe())) for out in (a, b)]
    for t in ts:
        t.start()
    s.thread.start()
    s.thread.join()
    for t in ts:
        t.join()
    assert a == b and a


def test_late_subscriber_gets_block_replay_only(oracle_engine, service_config):
    s = _finished(SessionManager(), with_fields(service_config, total_frames=15), "p")
    docs = [json.loads(l) for l in s.log.subscribe()]
    assert [d["index"] for d in docs] == list(range(5))
    assert all(d["type"] == "block" for d in docs)


def test_mid_run_subscriber_replays_then_tails(oracle_engine, service_config):
    m = SessionManager()
    s = m.create(service_config, "p", pace_seconds=0.01)
    while s.blocks_emitted < 5:
        time.sleep(0.005)
    docs = [json.loads(l) for l in s.log.subscribe()]
    s.thread.join()
    assert [d["index"] for d in docs if d["type"] == "block"] == list(range(13))
    assert docs[0]["type"] == "block" and docs[-1]["type"] == "done"


def test_failed_session_reports_error(oracle_engine, service_config, monkeypatch):
    from paper_2511_20426_b200 import service

    def boom(*a, **k):
        raise RuntimeError("device lost")
    monkeypatch.setattr(service, "run_cascade", boom)
    s = SessionManager().create(service_config, "p")
    s.thread.join()
    assert s.snapshot()["status"] == "failed" and "device lost" in s.snapshot()["error"]
    assert list(s.log.subscribe()) == []


def _sse(lines):
    for raw in lines:
        if raw.startswith("data: "):
            yield json.loads(raw[len("data: "):])


def test_http_routes(oracle_engine):
    from fastapi.testclient import TestClient
    c = TestClient(create_app())
    r = c.post("/sessions", json={"prompt": "a red cube", "config": {"total_frames": 15, "workers": 1}})
    assert r.status_code == 201
    sid = r.json()["id"]
    events = []
    with c.stream("GET", f"/sessions/{sid}/events") as st:
        for doc in _sse(st.iter_lines()):
            events.append(doc)
            if doc["type"] == "done":
                break
    assert [e["index"] for e in events if e["type"] == "block"] == list(range(5))
    for _ in range(200):
        snap = c.get(f"/sessions/{sid}").json()
        if snap["status"] == "done":
            break
        time.sleep(0.01)
    assert snap["status"] == "done" and snap["blocks_emitted"] == 5
    # invalid config -> 400 with the offending fields
    r = c.post("/sessions", json={"prompt": "x", "config": {"window_blocks": 2, "offset": 1}})
    assert r.status_code == 400 and "offset" in r.json()["detail"]["fields"]
    # unknown session -> 404
    assert c.get("/sessions/nope").status_code == 404
    assert c.post("/sessions/nope/prompt", json={"prompt": "x"}).status_code == 404
    # switch after the end -> 409
    assert c.post(f"/sessions/{sid}/prompt", json={"prompt": "y", "mode": "cascade"}).status_code == 409
    # distinct ids for identical requests
    body = {"prompt": "x", "config": {"total_frames": 3}}
    assert c.post("/sessions", json=body).json()["id"] != c.post("/sessions", json=body).json()["id"]


def test_live_switch_ack_carries_boundary(oracle_engine):
    from fastapi.testclient import TestClient
    c = TestClient(create_app())
    sid = c.post("/sessions", json={"prompt": "first", "config": {"total_frames": 39, "workers": 1},
                                    "pace_seconds": 0.01}).json()["id"]
    ack = c.post(f"/sessions/{sid}/prompt", json={"prompt": "second", "mode": "cascade"})
    assert ack.status_code == 200
    d = ack.json()
    assert d["extra_passes"] == 0 and d["mode"] == "cascade" and 0 <= d["boundary_block"] < 13


@pytest.mark.gpu
def test_device_engine_session_stream():
    """The service driving the device engine (toy model, fp64 on the GPU):
    the live stream equals the replay of the session's own trace."""
    m = SessionManager()
    cfg = CascadeConfig(total_frames=39, workers=2, pass_cost_base=1.0)
    s = m.create(cfg, "a red cube", start=False)
    got = []
    t = threading.Thread(target=lambda: got.extend(s.log.subscribe()))
    t.start()
    s.thread.start()
    s.thread.join()
    t.join()
    assert s.status == "done", s.error
    assert got == events_from_trace(s.result.trace, cfg, s.result.outputs)
    assert sum(json.loads(l)["type"] == "block" for l in got) == 13
