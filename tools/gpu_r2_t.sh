#!/bin/bash
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do timeout 300 python tools/theta_scan.py dpp - 2>&1 | tail -1; done
timeout 300 python tools/theta_scan.py peierls - 2>&1 | tail -1
