"""Print the composite-pair loop body (VOTE.ANY .. VOTE.ANY around the first
iteration holding two expf evaluations) of a SASS dump, with a count."""
import re, sys
lines = [re.sub(r"/\*[^*]*\*/", "", l).strip() for l in open(sys.argv[1])]
lines = [l for l in lines if l and not l.startswith(".")]
votes = [i for i, l in enumerate(lines) if "VOTE.ANY" in l]
for a, b in zip(votes, votes[1:]):
    body = lines[a + 1:b + 2]
    if sum("6.75539944105574400000e+15" in l and "DFMA" in l for l in body) >= 2 and \
            not any("CALL" in l for l in body):
        for l in body:
            print(l)
        ins = [l for l in body if not l.startswith("BRA.DIV")]
        print("instructions:", len(body), {k: sum(k in l for l in body) for k in ("LDC", "LDS", "DFMA", "DADD", "DMUL", "F2F", "MOV", "IMAD", "LOP3")})
        break
