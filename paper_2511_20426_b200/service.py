"""Streaming session service fed by the device engine.

The reference's gateway (``gateway.py:135-360``) runs ``run_cascade`` in a
daemon thread per session, projects every trace event into JSON lines
(``stream.TraceProjector``, byte-identical to the reference's) and serves
them as server-sent events, with a replay of the block events for
subscribers that join late.  This module offers the same interface --
``EventLog.publish / close / subscribe``, ``SessionManager.create / get /
switch``, ``Session.snapshot`` and the FastAPI routes of ``create_app``
(``POST /sessions``, ``GET /sessions/{id}``, ``POST /sessions/{id}/prompt``,
``GET /sessions/{id}/events``) with the same status codes -- around the
B200 engine: the session thread drives the device iterations and each
iteration's lines are published the moment its ``event_sink`` fires.

The log is one shared, append-only list guarded by a condition variable;
every subscriber keeps only a cursor into it (no per-subscriber copies).
A subscriber that joins at line k first receives the block lines among
lines[0:k] (the reference's bounded replay: a late joiner sees every block
but not the old metrics), then every line from k on.
"""

from __future__ import annotations

import json
import threading
import uuid

from .config import CascadeConfig, config_from_mapping
from .engine import DEFAULT_SESSION_SEED, DEFAULT_WEIGHT_SEED, run_cascade
from .errors import InvalidInputError
from .interactive import CommandQueue, LiveSwitchRequest
from .stream import TraceProjector

STATUS_RUNNING = "running"
STATUS_DRAINING = "draining"
STATUS_DONE = "done"
STATUS_FAILED = "failed"

_WAIT_SLICE = 0.5    # seconds a subscriber sleeps between checks for new lines


class EventLog:
    """Append-only line log: live fan-out plus block replay for late joiners."""

    def __init__(self):
        self._cv = threading.Condition()
        self._lines: list[str] = []
        self._is_block: list[bool] = []
        self._closed = False

    def publish(self, line: str) -> None:
        kind = json.loads(line).get("type")
        with self._cv:
            self._lines.append(line)
            self._is_block.append(kind == "block")
            self._cv.notify_all()

    def close(self) -> None:
        with self._cv:
            self._closed = True
            self._cv.notify_all()

    @property
    def closed(self) -> bool:
        with self._cv:
            return self._closed

    def subscribe(self):
        """Generator: replayed block lines, then the live tail until closed."""
        with self._cv:
            cursor = len(self._lines)
            head = [ln for ln, blk in zip(self._lines[:cursor], self._is_block) if blk]
        yield from head
        while True:
            with self._cv:
                while cursor == len(self._lines) and not self._closed:
                    self._cv.wait(_WAIT_SLICE)
                chunk = self._lines[cursor:]
                cursor += len(chunk)
                finished = self._closed and cursor == len(self._lines)
            yield from chunk
            if finished:
                return


class Session:
    """One generation session: its config, log, live-command queue and the
    thread driving the device engine."""

    def __init__(self, config: CascadeConfig, prompt: str, session_seed: int, weight_seed: int):
        self.id = uuid.uuid4().hex
        self.config, self.prompt = config, prompt
        self.session_seed, self.weight_seed = session_seed, weight_seed
        self.log = EventLog()
        self.queue = CommandQueue()
        self.status = STATUS_RUNNING
        self.error = None
        self.blocks_emitted = 0
        self.thread = None
        self.result = None

    def snapshot(self) -> dict:
        return {"id": self.id, "status": self.status, "prompt": self.prompt,
                "blocks_emitted": self.blocks_emitted, "total_blocks": self.config.num_blocks,
                "error": self.error}


class SessionManager:
    """Registry of sessions; each runs in its own daemon thread."""

    def __init__(self, weights=None, device: int | None = None):
        self._mu = threading.Lock()
        self._by_id: dict[str, Session] = {}
        self._weights = weights          # optional shared device weights (e.g. a Wan model)
        self._device = device

    def create(self, config: CascadeConfig, prompt: str, session_seed: int = DEFAULT_SESSION_SEED,
               weight_seed: int = DEFAULT_WEIGHT_SEED, pace_seconds: float = 0.0,
               start: bool = True) -> Session:
        config.validate()
        if not prompt:
            raise InvalidInputError("prompt must be a non-empty string", fields=["prompt"])
        s = Session(config, prompt, session_seed, weight_seed)
        proj = TraceProjector(config, weight_seed=weight_seed)
        drain_from = (config.num_blocks - 1) * config.offset

        def on_event(event, latents):
            for line in proj.feed(event, latents):
                s.log.publish(line)
            if event.emitted_block is not None:
                s.blocks_emitted += 1
            s.status = STATUS_DRAINING if event.iteration >= drain_from else STATUS_RUNNING

        def drive():
            try:
                if self._device is not None:
                    import torch
                    torch.cuda.set_device(self._device)
                s.result = run_cascade(config, prompt, session_seed=session_seed, weight_seed=weight_seed,
                                       command_queue=s.queue, event_sink=on_event,
                                       pace_seconds=pace_seconds, weights=self._weights)
                s.log.publish(proj.finish(s.result.trace))
                s.status = STATUS_DONE
            except Exception as exc:      # reported through the status route
                s.status = STATUS_FAILED
                s.error = str(exc)
                s.queue.reject_all(exc)
            finally:
                s.log.close()

        s.thread = threading.Thread(target=drive, name=f"session-{s.id[:8]}", daemon=True)
        with self._mu:
            self._by_id[s.id] = s
        if start:
            s.thread.start()
        return s

    def get(self, session_id: str) -> Session:
        with self._mu:
            s = self._by_id.get(session_id)
        if s is None:
            raise KeyError(session_id)
        return s

    def switch(self, session_id: str, prompt: str, mode: str):
        s = self.get(session_id)
        if s.status in (STATUS_DONE, STATUS_FAILED):
            raise InvalidInputError("session already finished")
        return s.queue.submit(LiveSwitchRequest(prompt, mode)).wait(timeout=60.0)


def create_app(manager: SessionManager | None = None):
    """FastAPI app with the reference's routes and status codes."""
    from fastapi import FastAPI, HTTPException
    from fastapi.responses import StreamingResponse

    app = FastAPI(title="blockcascade-b200")
    app.state.manager = manager or SessionManager()

    def lookup(session_id: str) -> Session:
        try:
            return app.state.manager.get(session_id)
        except KeyError:
            raise HTTPException(status_code=404, detail=f"unknown session {session_id}")

    def bad_input(exc: InvalidInputError, status: int = 400):
        return HTTPException(status_code=status, detail={"error": str(exc), "fields": exc.fields})

    @app.post("/sessions", status_code=201)
    def post_session(body: dict):
        try:
            cfg = (config_from_mapping(body["config"]) if body.get("config")
                   else getattr(app.state, "default_config", None) or CascadeConfig())
            s = app.state.manager.create(
                cfg, body.get("prompt", ""),
                session_seed=int(body.get("session_seed", DEFAULT_SESSION_SEED)),
                weight_seed=int(body.get("weight_seed", DEFAULT_WEIGHT_SEED)),
                pace_seconds=float(body.get("pace_seconds", getattr(app.state, "pace_seconds", 0.0))))
        except InvalidInputError as exc:
            raise bad_input(exc)
        return {"id": s.id}

    @app.get("/sessions/{session_id}")
    def get_session(session_id: str):
        return lookup(session_id).snapshot()

    @app.post("/sessions/{session_id}/prompt")
    def post_prompt(session_id: str, body: dict):
        s = lookup(session_id)
        try:
            ev = app.state.manager.switch(s.id, body.get("prompt", ""), body.get("mode", "cascade"))
        except InvalidInputError as exc:
            raise bad_input(exc, 409 if "finished" in str(exc) else 400)
        return ev.to_dict()

    @app.get("/sessions/{session_id}/events")
    def get_events(session_id: str):
        s = lookup(session_id)
        return StreamingResponse((f"data: {line}\n\n" for line in s.log.subscribe()),
                                 media_type="text/event-stream")

    return app
