for prs in 2 4 8; do for cw in CW4 CW8; do
  for st in 1 3; do echo "prs=$prs $cw streams=$st"; env BITEDGE_PRS=$prs BITEDGE_$cw=1 KB_STREAMS=$st timeout 60 python scripts/kbench.py c3; done
done; done
