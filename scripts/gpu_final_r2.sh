#!/bin/bash
# round-2 final: GPU tests, default bench, reference arm, then the profiles
bash scripts/gpu_r2.sh
bash scripts/gpu_profiles_r2.sh
