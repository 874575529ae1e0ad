"""Run a child command in its own process group and, on timeout, kill that whole group (torchrun's
worker ranks included), so a stuck multi-process run never outlives its test holding the GPU."""

import os
import signal
import subprocess


def run_group(cmd, timeout, **kw):
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, start_new_session=True, **kw)
    try:
        out, err = p.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, signal.SIGKILL)  # the group this call created, nothing else
        out, err = p.communicate()
        err = (err or "") + f"\n[run_group] killed after {timeout} s"
    return subprocess.CompletedProcess(cmd, p.returncode, out, err)
