for cfg in "1.1 3" "1.1 2" "1.1 4" "1.1 6"; do set -- $cfg; echo "thresh $1 div $2"; NT_ATTN_SPLIT_THRESH=$1 NT_ATTN_SPLIT_DIV=$2 python tools/split_probe.py; done
