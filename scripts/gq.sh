#!/bin/bash
# build locally, then run the quick GPU script only if the build is clean
make -j16 lib >/tmp/build.log 2>&1 || { grep -E "error" -A3 /tmp/build.log | head -20; exit 1; }
timeout 2400 /usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-1200} -- "$@" 2>&1 | tail -${TAILN:-4} | cut -c1-${CUTN:-1800}
