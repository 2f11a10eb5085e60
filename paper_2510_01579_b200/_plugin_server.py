"""Kernel-plugin server for workers forked after CUDA was initialised.

A process forked from a parent that had initialised CUDA cannot use CUDA
itself.  The reference's harness forks its worker pools
(harness/workers.py:36-38) after the parent may already have run the plugin,
so ``_kernel_cuda.run_anneals`` in such a worker forwards the call here: one
server per worker, started with exec (``python -m
paper_2510_01579_b200._plugin_server``, a fresh process with its own CUDA
context), serving ``run_anneals`` requests over its stdin/stdout as pickled
tuples.  The server runs the same FP64-exact kernel, so the outputs are the
ones the worker would have computed itself.  It exits when the worker closes
the pipe (worker exit included).
"""

from __future__ import annotations

import os
import pickle
import struct
import subprocess
import sys
import threading

_HDR = struct.Struct("<Q")


def _send(f, obj) -> None:
    data = pickle.dumps(obj, protocol=pickle.HIGHEST_PROTOCOL)
    f.write(_HDR.pack(len(data)))
    f.write(data)
    f.flush()


def _recv(f):
    hdr = f.read(_HDR.size)
    if len(hdr) < _HDR.size:
        raise EOFError
    (n,) = _HDR.unpack(hdr)
    data = f.read(n)
    if len(data) < n:
        raise EOFError
    return pickle.loads(data)


class _Client:
    def __init__(self):
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        env = dict(os.environ)
        env["PYTHONPATH"] = root + os.pathsep + env.get("PYTHONPATH", "")
        self.proc = subprocess.Popen([sys.executable, "-m", "paper_2510_01579_b200._plugin_server"],
                                     stdin=subprocess.PIPE, stdout=subprocess.PIPE, env=env,
                                     close_fds=True)
        self.lock = threading.Lock()
        self.pid = os.getpid()

    def run_anneals(self, *args):
        with self.lock:
            _send(self.proc.stdin, ("run_anneals", args))
            ok, out = _recv(self.proc.stdout)
        if not ok:
            exc_type, msg = out
            raise (ValueError if exc_type == "ValueError" else RuntimeError)(msg)
        return out


_client = None
_client_lock = threading.Lock()


def client() -> _Client:
    """The calling process's server (started on first use)."""
    global _client
    with _client_lock:
        if _client is None or _client.pid != os.getpid() or _client.proc.poll() is not None:
            _client = _Client()
        return _client


def serve(fin, fout) -> None:
    from . import _kernel_cuda
    while True:
        try:
            name, args = _recv(fin)
        except EOFError:
            return
        try:
            if name != "run_anneals":
                raise ValueError(f"unknown request {name!r}")
            _send(fout, (True, _kernel_cuda.run_anneals(*args)))
        except Exception as e:  # errors travel back to the caller
            _send(fout, (False, (type(e).__name__, str(e))))


if __name__ == "__main__":
    # the protocol owns the original stdout; anything else printed to fd 1
    # (library diagnostics) goes to stderr
    proto = os.fdopen(os.dup(1), "wb")
    os.dup2(2, 1)
    serve(sys.stdin.buffer, proto)
