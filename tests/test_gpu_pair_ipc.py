"""MPC_MODE_PAIR across two processes: party 0 and party 1 in separate processes
exchange every opening through cudaIpc-mapped peer memory -- the remote path bench.py takes for
N > 1 -- and every op's output shares equal MPC_MODE_BOTH's bit for bit (tools/pair_ipc_check.py;
on a one-GPU box both processes share cuda:0)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("exchange", [1, 0])      # LL63 (the MPC_MODE_PAIR default) and LL
def test_pair_two_processes_bit_identical_to_both(exchange):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "pair_ipc_check.py"), f"--exchange={exchange}"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "PAIR_IPC_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_pair_debug_header_detects_mismatched_calls():
    """mpc_ctx_set_debug: party 0 issues mul while party 1 issues square; both contexts report
    MPC_ERR_PROTOCOL at sync."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "pair_ipc_check.py"), "--mismatch"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "PAIR_IPC_PROTOCOL_DETECTED" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_pair_two_processes_party1_without_k0_reads_the_dealer_stream():
    """party 1's context is created with key_p0 = 0 and reads its correction words
    from an MPC_MODE_DEALER context's offline stream; every op's shares still equal MPC_MODE_BOTH's."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "pair_ipc_check.py"), "--dealer"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "PAIR_IPC_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
