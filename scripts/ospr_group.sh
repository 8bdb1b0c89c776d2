#!/bin/bash
for g in 64 12 8 4 2 1; do
  echo "group $g: 2048 $(CGHB200_OSPR_GROUP=$g python scripts/prof_ospr.py 2048 24 2>&1 | tail -1 | cut -c1-40)  1024 $(CGHB200_OSPR_GROUP=$g python scripts/prof_ospr.py 1024 24 2>&1 | tail -1 | cut -c1-40)"
done
