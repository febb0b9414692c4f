// Device-side encoding of a compiled rewrite program (the reference's
// DispatchTable, proj/include/trs/dispatch.hpp:73-78), packed into one blob
// that every CTA of the step loop copies into shared memory.
//
// Besides the reference fields, each rule carries the *subscription plan*
// of its RHS template: which freshly built node waits on which other fresh
// node.  A constructive rewrite at sweep s writes nodes that the reference
// would first inspect at sweep s+1, where every bound-variable child is
// already nf and every fresh child is not; so each fresh
// node's first fresh child (in argument order) is exactly the child its
// sweep-(s+1) subterm scan (sweep_engine.cpp:173-178) stops on.  The engine
// records that wait at build time instead of re-discovering it one sweep
// later.  Nodes with no fresh child go on the next sweep's frontier list.
#pragma once

#include <cstdint>

namespace trs_b200 {

constexpr uint32_t kSymBits = 24;
constexpr uint32_t kSymMask = (1u << kSymBits) - 1;
constexpr uint32_t kDeadHead = 0xFFFFFFFFu;  // head word of a collected slot
constexpr uint32_t kWoken = 0xFFFFFFFFu;     // waiter word: node is nf, do not sleep on it
constexpr uint8_t kNone = 0xFF;
constexpr uint8_t kRootSub = 0xFE;

constexpr uint32_t kMaxRuleSteps = 48;
constexpr uint32_t kMaxRuleInstrs = 32;
constexpr uint32_t kMaxVars = 16;
constexpr uint32_t kMaxProgramBytes = 40 * 1024;

// record word layout (W words per slot, W = 8/16/32):
//   w0 head = symbol | subterm cursor << 24
//   w1 nf epoch (sweep in which the slot became nf; 0 = not nf)
//   w2 refcount
//   w3 waiter (slot of the parent sleeping on this one, 0 none, kWoken)
//   w4.. arguments
constexpr uint32_t kWHead = 0, kWEpoch = 1, kWRc = 2, kWWaiter = 3, kWArgs = 4;

struct DRule {
    uint16_t first_step;
    uint8_t num_steps;
    uint8_t num_vars;
    uint16_t first_instr;
    uint8_t num_instrs;
    uint8_t new_slots;
    uint16_t root_ref;   // bit 15: node ref, else var slot
    uint8_t collapse;
    uint8_t root_wait;   // fresh instr the rewritten root sleeps on (kNone: push root)
    uint8_t root_cursor; // argument position of that wait
    uint8_t pad[3];
    uint32_t push_mask;  // bit k: fresh instr k goes on the next frontier list
};
static_assert(sizeof(DRule) == 20, "DRule layout");

struct DStep {
    uint8_t kind;  // 0 CheckHead, 1 BindVar
    uint8_t child;
    int8_t parent; // step index within the rule, -1 = redex root
    uint8_t pad;
    uint32_t value;
};
static_assert(sizeof(DStep) == 8, "DStep layout");

struct DInstr {
    uint32_t symbol;
    uint16_t first_ref;
    uint8_t indegree;
    uint8_t subscriber;  // who sleeps on this fresh node: kNone, kRootSub or instr index
    uint8_t cursor;      // argument position this node itself waits at
    uint8_t pad[3];
};
static_assert(sizeof(DInstr) == 12, "DInstr layout");

constexpr uint16_t kRefNode = 0x8000;

struct ProgHeader {
    uint32_t num_symbols;
    uint32_t num_rules;
    uint32_t num_steps;
    uint32_t num_instrs;
    uint32_t num_refs;
    uint32_t max_arity;
    uint32_t max_new_slots;
    uint32_t off_arity;       // uint8_t[num_symbols]
    uint32_t off_rule_begin;  // uint16_t[num_symbols + 1]
    uint32_t off_rules;       // DRule[]
    uint32_t off_steps;       // DStep[]
    uint32_t off_instrs;      // DInstr[]
    uint32_t off_refs;        // uint16_t[]
    uint32_t bytes;           // total blob size (multiple of 16)
};

}  // namespace trs_b200
