#!/bin/bash
# build the library; print warnings/errors; exit non-zero on failure
out=$(make -C /root/repo/paper_2603_24919_b200/csrc -j8 2>&1); rc=$?
echo "$out" | grep -E "error|warning" | head -5
exit $rc
