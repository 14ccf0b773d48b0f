#!/bin/bash
timeout 300 python scripts/attn_ab.py scratch/new3.so scratch/base.so 2>&1 | tail -4
timeout 300 python scripts/attn_ab.py scratch/base.so scratch/new3.so 2>&1 | tail -4
