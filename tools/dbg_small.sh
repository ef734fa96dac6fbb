#!/bin/bash
# quick hang/parity probe of the scan kernel on tiny inputs (each under its own timeout)
timeout 120 python tools/dbg_fast.py 2>&1 | tail -12; echo dbg=$?
