#!/bin/bash
# long whole-frame runs (measured seconds per frame) -> profiles/*_frames_r02*.json
mkdir -p gpurun_out/frames
for spec in "$@"; do
  set -- $spec
  name=$1; shift
  echo "== $name: $*" >> gpurun_out/frames/frames.log
  timeout ${FRAME_TIMEOUT:-1500} python tools/c4_frames.py "$@" --out gpurun_out/frames/$name.json >> gpurun_out/frames/frames.log 2>&1
  echo "rc=$?" >> gpurun_out/frames/frames.log
done
tail -5 gpurun_out/frames/frames.log
