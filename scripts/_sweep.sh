cd $GRAFT_REPO_ROOT
LIBF=paper_2407_11550_b200/lib/libadakv_b200.so
cp var/w4.so $LIBF
ADAKV_DECODE_CS=16 timeout 60 python scripts/dec_ts4.py 2>&1 | grep -v NCCL | sed -n '1,4p;14,60p'
cp var/base.so $LIBF
