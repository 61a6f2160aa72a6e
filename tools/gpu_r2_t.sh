#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/theta_scan.py dpp - gj_pair=3 gj_pair=1 2>&1 | tail -3
